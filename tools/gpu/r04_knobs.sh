# same-call knob sweep after the slicer / generator trims: scanners 2, GEN8 16, TEAMS2 2, no sleep, sleep 30 ns, first sub-chunk 32 steps
for cfg in "1000000 128 256" "4194304 64 128" "4000000 256 512" "1000000 512 768"; do
  timeout 120 python tools/sk_time.py $cfg
  for v in s2 g8 tm2 sl0 sl30 sf32; do CQR_LIB=tools/gpu/libcqr_$v.so timeout 120 python tools/sk_time.py $cfg; done
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_knobs.txt
