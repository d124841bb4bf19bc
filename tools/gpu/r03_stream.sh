timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stream_ordered or cholqr_family" > gpurun_out/pt_stream.log 2>&1; tail -3 gpurun_out/pt_stream.log
python tools/gpu/overhead2.py
