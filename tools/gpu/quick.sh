# GPU tests + one c1 pipeline run + launch list of the c1 kernels
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_quick.log 2>&1; tail -2 gpurun_out/pt_quick.log
python tools/prof_c1.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_quick.csv python tools/prof_c1.py > /dev/null 2>&1
python3 -c "
import sys; sys.path.insert(0,'tools')
import ncu_summary as s
for k,v in s.launches('gpurun_out/launches_quick.csv')[-16:]: print(f'{v:10.1f} us  {k[:70]}')
"
