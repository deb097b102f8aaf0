for rep in 1 2; do for lib in variants/libhc_nraw2.so variants/libhc_nraw1.so; do
  echo "$lib: $(HC_LIB=$lib timeout 200 python tools/quick_time.py c4 c3 c2 | tr '\n' ' ')"
done; done
for lib in paper_1608_00206_b200/libhc.so variants/libhc_nraw2.so; do
  HC_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:slab8 -s 1 -c 1 python tools/quick_time.py c4 2>&1 | grep -E "dram__|lts__|l1tex|issue" | sed "s|^|$(basename $lib) |"
done
