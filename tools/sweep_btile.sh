# dev: timing experiment, half of each register-tile inverse loaded (wrong results)
MODES=btile@reg python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply"
BD_EXP_HALF=1 MODES=btile@reg python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply"
