# what the ring alone costs (no slicing, no scan, no draws): p0 = ring, p1 = + no MMAs, p2 = + no Omega digit stores,
# p3 = + no A loads, p4 = + no proxy fence in the generators, p5 = p2 + p3 + p4
for cfg in "4194304 64 128" "1000000 128 256" "4000000 256 512"; do
  for v in p0 p1 p2 p3 p4 p5; do CQR_LIB=tools/gpu/libcqr_$v.so timeout 120 python tools/sk_time.py $cfg; done
done 2>&1 | grep "sketch\|rror" | tee gpurun_out/r04_ring.txt
