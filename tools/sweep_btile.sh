# dev sweep of triangular-solve kernel knobs on cfg2 (fwd+bwd pair, median of 30)
MODES=btile@smem,btile@reg,btile@regt,btile@pipe python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|rel diff|Error|error"
BD_BTILE_KERNEL=regt python tools/btile_trace.py 128,128,64 2 2>&1 | grep -v "^\[bd\]"
KERNELS="reg regt" bash tools/sweep_bench.sh
