# Omega ring / A-plane ring / FP64 A ring depths: main (S,P,AS as before) vs v532, v523; accuracy check of each
for cfg in "1000000 128 256" "4000000 256 512" "4194304 64 128" "1000000 512 768"; do
  for v in "" v532 v523; do
    if [ -z "$v" ]; then timeout 120 python tools/sk_time.py $cfg; else CQR_LIB=tools/gpu/libcqr_$v.so timeout 120 python tools/sk_time.py $cfg; fi
  done
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_stages.txt
for v in v532 v523; do CQR_LIB=tools/gpu/libcqr_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "sketch" 2>&1 | tail -2; done | tee -a gpurun_out/r04_stages.txt
