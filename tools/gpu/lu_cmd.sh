# LU: parity tests, then the c1 launch list of the small kernels
timeout 600 python -m pytest tests -m gpu -x -q -k "lu or rlu or chol or breakdown" > gpurun_out/pt_lu.log 2>&1; tail -2 gpurun_out/pt_lu.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lu.csv python tools/prof_c1.py > /dev/null 2>&1
python3 -c "
import sys; sys.path.insert(0,'tools')
import ncu_summary as s
for k,v in s.launches('gpurun_out/launches_lu.csv')[-16:]:
  if any(x in k for x in ('lu_','chol')): print(f'{v:10.1f} us  {k[:60]}')
"
