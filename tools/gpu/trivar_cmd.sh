# trisolve variants: parity (trisolve / CholQR family bitwise) and per-width timings
for v in ${LIBS:-default}; do
  if [ "$v" = default ]; then unset CQR_LIB; else export CQR_LIB=tools/gpu/libcqr_$v.so; fi
  r=$(timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "trisolve or cholqr_family or rlu_uniform" 2>&1 | tail -1)
  echo "$v | $r"
  for n in ${NS:-128 256 512}; do PROF_N=$n timeout 120 python tools/prof_tri.py 2>&1 | tail -1 | sed "s/^/$v /"; done
done
