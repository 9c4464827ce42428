# dev: smem-staged register tiles at 8 CTAs/SM vs the register kernel across sizes
MODES=btile@reg,btile@rsmem python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply"
MODES=btile@reg,btile@rsmem python tools/trsv_bench.py 160,160,80 20 2>&1 | grep -E "us per apply"
MODES=btile@reg python tools/trsv_bench.py 192,192,96 10 2>&1 | grep -E "us per apply"
