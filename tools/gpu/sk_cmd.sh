# sketch probes: draw accuracy, then the c1 sketch timing for each library variant
timeout 300 python -m pytest tests -m gpu -x -q -k "gauss or sketch or rqr or rlu" > gpurun_out/pt_sk.log 2>&1; tail -2 gpurun_out/pt_sk.log
timeout 120 python tools/gpu/bm_acc.py
for v in ${LIBS:-default}; do
  if [ "$v" = default ]; then unset CQR_LIB; else export CQR_LIB=tools/gpu/libcqr_$v.so; fi
  for n in ${NS:-128}; do PROF_N=$n timeout 120 python tools/prof_sketch.py 2>&1 | tail -1 | sed "s/^/$v /"; done
done
