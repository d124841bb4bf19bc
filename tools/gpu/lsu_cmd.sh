# 8-column TMA boxes (conflict-free fragment loads) vs the previous 16-column swizzled boxes
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gram or sketch or gauss or rqr or rlu or cholqr" 2>&1 | tail -1
for v in default old; do
  if [ "$v" = default ]; then unset CQR_LIB; else export CQR_LIB=tools/gpu/libcqr_$v.so; fi
  for n in 128 256 512; do PROF_N=$n timeout 120 python tools/prof_gram.py 2>&1 | tail -1 | sed "s/^/$v /"; done
  for n in 64 128 256; do PROF_N=$n timeout 120 python tools/prof_sketch.py 2>&1 | tail -1 | sed "s/^/$v /"; done
done
