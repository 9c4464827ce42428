# Round GPU batch: full GPU tests, bench line, ncu launch list, ncu full capture
# of the default triangular-solve kernel (each profiler run after its command
# has exited 0 without ncu).  Outputs under gpurun_out/.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
BD_NO_GRAPH=1 python tools/profile_step.py --steps 1 > gpurun_out/profile_step.log 2>&1 && \
BD_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none -s 1000 -c 420 --csv \
  --log-file gpurun_out/launches.csv python tools/profile_step.py --steps 1 > gpurun_out/ncu_launch.log 2>&1
BD_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_trsv_rtile -s 600 -c 6 \
  -o gpurun_out/r01_rtile_full -f python tools/profile_step.py --steps 1 > gpurun_out/ncu_full.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
