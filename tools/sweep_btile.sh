# dev: register-tile occupancy at cfg2 and cfg3 sizes
MODES=btile@reg,btile@rsmem python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply"
MODES=btile@reg,btile@rsmem python tools/trsv_bench.py 256,256,128 10 2>&1 | grep -E "us per apply"
