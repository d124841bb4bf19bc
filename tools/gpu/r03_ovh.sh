CQR_TRACE=1 python tools/gpu/trace_call.py > gpurun_out/trace2.log 2>&1; tail -3 gpurun_out/trace2.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x > gpurun_out/pt_ovh.log 2>&1; tail -2 gpurun_out/pt_ovh.log
python tools/gpu/overhead2.py
