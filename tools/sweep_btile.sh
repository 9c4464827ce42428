# dev sweep of triangular-solve kernel knobs on cfg2 (fwd+bwd pair, median of 30)
run() { echo "== $*"; env "$@" MODES=btile python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff|Error|error"; }
run BD_BTILE_KERNEL=warp
run BD_BTILE_KERNEL=warp BD_BTILE_SLEEP=256
run BD_BTILE_KERNEL=warp BD_BTILE_SLEEP=1024
run BD_BTILE_KERNEL=warp BD_BTILE_PERSM=6
run BD_BTILE_KERNEL=warp BD_BTILE_PERSM=8 BD_BTILE_SLEEP=256
BD_BTILE_KERNEL=warp python tools/btile_trace.py 128,128,64 1 2>&1 | grep -v "^\[bd\]"
