for w in c2 c3 c4; do
  python tools/prof_one.py $w > /dev/null 2>&1 && ncu --profile-from-start off --set full --clock-control none \
    -k regex:"sketch_i8|trisolve|gram_leaf|panel_update|qr_blocked|lu_rot|chol|qr_warp" -c 10 -o /tmp/full_r03_$w python tools/prof_one.py $w > /tmp/ncu_full_r03_$w.log 2>&1; tail -1 /tmp/ncu_full_r03_$w.log
  python tools/ncu_summary.py full /tmp/full_r03_$w.ncu-rep > gpurun_out/r03_ncu_full_$w.txt 2>&1
done
