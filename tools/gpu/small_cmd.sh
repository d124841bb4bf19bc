timeout 600 python -m pytest tests -m gpu -x -q -k "lu or chol or rlu or rqr" > gpurun_out/pt_small.log 2>&1; tail -2 gpurun_out/pt_small.log
for v in 0 1; do
CQR_LU_VARIANT=$v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python tools/prof_c1.py > /dev/null 2>&1
python3 -c "
import sys; sys.path.insert(0,'tools')
import ncu_summary as s
for k,v in s.launches('gpurun_out/launches_small.csv')[-16:]:
  if any(x in k for x in ('lu_','chol','reduce','combine')): print(f'v$v {v:10.1f} us  {k[:60]}')
"
done
