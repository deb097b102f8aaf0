for lib in paper_1608_00206_b200/libhc.so variants/libhc_p2ch1.so; do
  echo "== $lib"; HC_LIB=$lib timeout 300 python tools/r02/t14.py 2>&1 | grep "D=1[4-7]"
done
