# same-call A/B: main vs tools/gpu/libcqr_prev.so, alternating, three rounds
for r in 1 2 3; do
  for cfg in "1000000 128 256" "4194304 64 128"; do
    timeout 120 python tools/sk_time.py $cfg; CQR_LIB=tools/gpu/libcqr_prev.so timeout 120 python tools/sk_time.py $cfg
  done
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_ab.txt
