# what bounds the i8 sketch: variants without the A slicers + scanners (nss), without the draws (ng), without either (nssg)
for cfg in "1000000 128 256" "4000000 256 512" "4194304 64 128" "1000000 512 768"; do
  for v in "" nss ng nssg; do
    if [ -z "$v" ]; then python tools/sk_time.py $cfg; else CQR_LIB=tools/gpu/libcqr_$v.so python tools/sk_time.py $cfg; fi
  done
done 2>&1 | grep sketch | tee gpurun_out/r04_probe.txt
