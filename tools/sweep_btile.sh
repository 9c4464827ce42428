# dev sweep of triangular-solve kernel knobs on cfg2 (fwd+bwd pair, median of 30)
run() { echo "== $*"; env "$@" MODES=btile python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff|Error|error"; }
MODES=btile@smem,btile@reg,btile@pipe python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff|Error|error"
run BD_BTILE_KERNEL=pipe BD_BTILE_PERSM=3
BD_BTILE_KERNEL=pipe python tools/btile_trace.py 128,128,64 2 2>&1 | grep -v "^\[bd\]"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
