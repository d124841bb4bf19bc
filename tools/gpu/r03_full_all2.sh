cap() {  # workload, kernel regex, tag
  python tools/prof_one.py $1 > /dev/null 2>&1 && ncu --profile-from-start off --set full --clock-control none -k regex:"$2" -c 1 \
    -o /tmp/f_$1_$3 python tools/prof_one.py $1 > /tmp/f_$1_$3.log 2>&1
  python tools/ncu_summary.py full /tmp/f_$1_$3.ncu-rep >> gpurun_out/r03_ncu_full_$1.txt 2>&1
}
for w in c2 c3 c4; do rm -f gpurun_out/r03_ncu_full_$w.txt; done
cap c2 sketch_i8 sk; cap c2 trisolve_tma tri; cap c2 gram_leaf_tma gram; cap c2 qr_blocked qr
cap c3 sketch_i8 sk; cap c3 trisolve_rr tri; cap c3 gram_leaf64 gram; cap c3 qr_warp qr
cap c4 sketch_i8 sk; cap c4 panel_update gemm; cap c4 trisolve_tma tri; cap c4 gram_leaf_tma gram
ls -la gpurun_out/r03_ncu_full_*.txt
