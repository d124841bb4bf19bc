# c3 (C = 1) generator teams 1 (main) / 2 / 4, and the select-free live mask (lf) at every config
for v in "" t2 t4 lf; do
  if [ -z "$v" ]; then timeout 120 python tools/sk_time.py 4194304 64 128; else CQR_LIB=tools/gpu/libcqr_$v.so timeout 120 python tools/sk_time.py 4194304 64 128; fi
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_teams.txt
for cfg in "1000000 128 256" "4000000 256 512" "1000000 512 768"; do
  for v in "" lf; do
    if [ -z "$v" ]; then timeout 120 python tools/sk_time.py $cfg; else CQR_LIB=tools/gpu/libcqr_$v.so timeout 120 python tools/sk_time.py $cfg; fi
  done
done 2>&1 | grep "sketch\|rror" | tee -a gpurun_out/r04_teams.txt
for v in t2 t4 lf; do CQR_LIB=tools/gpu/libcqr_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sketch" 2>&1 | tail -2; done | tee -a gpurun_out/r04_teams.txt
