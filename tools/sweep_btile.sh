# dev: automatic kernel choice at cfg2 and cfg3 sizes
BD_DEBUG=1 MODES=btile python tools/trsv_bench.py 128,128,64 30 2>&1 | grep -E "us per apply|auto"
BD_DEBUG=1 MODES=btile python tools/trsv_bench.py 256,256,128 10 2>&1 | grep -E "us per apply|auto"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize_cfg4.py -x -q 2>&1 | tail -2
python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
