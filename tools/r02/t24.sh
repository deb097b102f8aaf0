# which phase needs the L1 share: pass 1 alone (HC_DEBUG_SKIP=1: no pass 2) and pass 2 alone (=2) at three carve-outs
for skip in 0 1 2; do for lib in paper_1608_00206_b200/libhc.so variants/libhc_co75.so variants/libhc_co100.so; do
  echo "skip=$skip $lib: $(HC_DEBUG_SKIP=$skip HC_LIB=$lib timeout 200 python tools/quick_time.py c4 | tail -1)"
done; done
