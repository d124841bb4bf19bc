# LU variants: c1 launch-list time of lu_rot per library
for v in ${LIBS:-default}; do
  if [ "$v" = default ]; then unset CQR_LIB; else export CQR_LIB=tools/gpu/libcqr_$v.so; fi
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_luv.csv python tools/prof_c1.py > /dev/null 2>&1
  python3 -c "
import sys; sys.path.insert(0,'tools')
import ncu_summary as s
for k,v in s.launches('gpurun_out/launches_luv.csv')[-16:]:
  if 'lu_' in k: print(f'$v {v:10.1f} us  {k[:60]}')
"
done
