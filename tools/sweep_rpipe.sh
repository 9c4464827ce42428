# dev sweep: TMA-ring register tiles (k_trsv_rpipe) vs the default on the cfg2 slab
for d in 2 3; do
  BD_RPIPE_DEPTH=$d BD_DEBUG=1 MODES=btile@reg,btile@rpipe python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff|btile launch" | sed "s/^/depth=$d /"
done
