# dev: 5x5x5 lattice tiles (128-row rtile, smem inverse) vs the 4x4x4 default
BD_DEBUG=1 MODES=btile python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|auto|btile n=|launch"
BD_BTILE_ROWS=125 BD_DEBUG=1 MODES=btile python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|auto|btile n=|launch|rel diff"
BD_BTILE_ROWS=125 BD_DEBUG=1 MODES=btile python tools/trsv_bench.py 256,256,128 10 2>&1 | grep -E "us per apply|btile n=|launch"
