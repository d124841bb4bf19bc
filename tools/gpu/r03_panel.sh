timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "trisolve" > gpurun_out/pt_panel.log 2>&1; tail -3 gpurun_out/pt_panel.log
for mn in "1000000 256" "1000000 512"; do
  CQR_TRISOLVE_VARIANT=2 python tools/tri_ab.py $mn
  CQR_TRISOLVE_VARIANT=0 python tools/tri_ab.py $mn
  CQR_TRISOLVE_NO_PANELS=1 CQR_TRISOLVE_VARIANT=np python tools/tri_ab.py $mn
done
