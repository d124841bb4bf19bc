timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sketch or gaussian" > gpurun_out/pt_i8.log 2>&1; tail -1 gpurun_out/pt_i8.log
for a in "1000000 128 256" "4000000 256 512" "4194304 64 128" "1000000 512 768"; do python tools/sk_time.py $a; done
