# Round GPU batch: full GPU tests, bench line, ncu launch list, ncu full capture
# of the default triangular-solve kernel (each profiler run after its command
# has exited 0 without ncu).  Outputs under gpurun_out/ (tag = $1, default r02).
TAG=${1:-r02}
set -x
python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
BD_NO_GRAPH=1 python tools/profile_step.py --steps 1 > gpurun_out/${TAG}_profile_step.log 2>&1 && \
BD_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --clock-control none -s 1000 -c 600 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py --steps 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
BD_NO_GRAPH=1 ncu --set full --clock-control none --import-source on -k regex:k_trsv_rpipe -s 600 -c 6 \
  -o gpurun_out/${TAG}_rpipe_full -f python tools/profile_step.py --steps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1
