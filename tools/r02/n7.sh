for lib in paper_1608_00206_b200/libhc.so variants/libhc_p2wb.so variants/libhc_p2el.so; do
  echo "$lib: $(HC_LIB=$lib timeout 200 python tools/quick_time.py c4 | tail -1)"
done
for lib in paper_1608_00206_b200/libhc.so variants/libhc_p2wb.so variants/libhc_p2el.so; do
  HC_LIB=$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:slab8 -s 1 -c 1 python tools/quick_time.py c4 2>&1 | grep -E "dram__|duration" | sed "s|^|$(basename $lib) |"
done
for lib in paper_1608_00206_b200/libhc.so variants/libhc_p2wb.so; do
  echo "$lib: $(HC_LIB=$lib timeout 200 python tools/quick_time.py c4 | tail -1)"
done
