# dev sweep: blocked-tile triangular-solve kernels (BD_BTILE_KERNEL) on the
# cfg2 slab and at cfg3 size (forward + backward pair, median of N reps)
MODES=btile@auto,btile@reg,btile@rsmem,btile@smem python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff"
MODES=btile@auto,btile@rsmem,btile@smem python tools/trsv_bench.py 256,256,128 10 2>&1 | grep -E "us per apply|rel diff"
