# Cholesky panel-width variants: parity (Cholesky / CholQR family bitwise tests) and the c1 Cholesky stage
for v in ${LIBS:-default}; do
  if [ "$v" = default ]; then unset CQR_LIB; else export CQR_LIB=tools/gpu/libcqr_$v.so; fi
  r=$(timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cholesky or cholqr or breakdown or scholqr" 2>&1 | tail -1)
  s=$(PROF_REPS=6 timeout 120 python tools/prof_c1.py 2>&1 | tail -1)
  echo "$v | $r | $s"
done
