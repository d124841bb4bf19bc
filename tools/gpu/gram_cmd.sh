timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_gram.log 2>&1; tail -2 gpurun_out/pt_gram.log
for n in 64 128 256; do PROF_N=$n python tools/prof_gram.py; CQR_GRAM_LEGACY=1 PROF_N=$n python tools/prof_gram.py | sed 's/^/legacy /'; done
