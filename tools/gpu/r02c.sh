for i in 1 2; do timeout 900 python -m pytest tests/test_gpu_configs.py tests/test_gpu_acceptance.py -m gpu -q -s > gpurun_out/pt_r02c_$i.log 2>&1; grep -E "FAIL|Error|passed|failed" gpurun_out/pt_r02c_$i.log | head; done
for i in 1 2 3; do python tools/gpu/debug_acc2.py 1 2 3 | grep -v "^done"; done
