# Round capture r04: GPU tests, smoke, bench lines c1-c4, per-config launch lists with DRAM bytes, ncu --set full of c1's top kernels
tag=${1:-r04}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; tail -2 gpurun_out/pytest_gpu_${tag}.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${tag}.log 2>&1; tail -1 gpurun_out/smoke_${tag}.log
python bench.py > gpurun_out/bench_${tag}_c1.json 2> gpurun_out/bench_${tag}_c1.err
for w in c2 c3 c4; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_${tag}_$w.json 2> gpurun_out/bench_${tag}_$w.err; done
for w in c1 c2 c3 c4; do
  python tools/prof_one.py $w > gpurun_out/prof_${tag}_$w.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${tag}_$w.csv python tools/prof_one.py $w > /dev/null 2>&1
done
python tools/prof_one.py c1 > /dev/null 2>&1 && ncu --profile-from-start off --set full --clock-control none \
    -k regex:"sketch_i8|trisolve_tma|gram_leaf|lu_rot|cholesky|panel_update" -c 8 -o /tmp/full_${tag}_c1 python tools/prof_one.py c1 > /tmp/ncu_full_${tag}.log 2>&1
tail -1 /tmp/ncu_full_${tag}.log
python tools/ncu_summary.py full /tmp/full_${tag}_c1.ncu-rep > gpurun_out/ncu_full_${tag}_c1.txt 2>&1
python -c "
import json
for w in ('c1','c2','c3','c4'):
    d = json.load(open('gpurun_out/bench_${tag}_%s.json' % w)); print(w, round(d['ms_per_step'], 3), round(d['value'], 2), {k: round(v, 3) for k, v in d['stage_ms'].items()})
"
for w in c2 c3 c4; do
  python tools/prof_one.py $w > /dev/null 2>&1 && ncu --profile-from-start off --set full --clock-control none \
    -k regex:"sketch_i8|trisolve|gram_leaf|panel_update|qr_warp|qr_blocked" -c 6 -o /tmp/full_${tag}_$w python tools/prof_one.py $w > /tmp/ncu_full_${tag}_$w.log 2>&1
  python tools/ncu_summary.py full /tmp/full_${tag}_$w.ncu-rep > gpurun_out/ncu_full_${tag}_$w.txt 2>&1
done
du -sh gpurun_out
