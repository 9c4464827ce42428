# exact-inner relaxed supernodes (BD_SUPER_RELAX) on config 1: dev ms/step
for r in ${RELAX:-0 0.4 0.5 0.6 0.7 0.8}; do
  BD_SUPER_RELAX=$r python tools/cfg_run.py --workload cfg1 --steps 25 > gpurun_out/rx_$r.log 2>&1
done
BD_SUPER_RELAX=${RELAX_TEST:-0.5} python -m pytest tests/test_gpu_trsv_variants.py -q -p no:cacheprovider -k exact > gpurun_out/rx_tests.log 2>&1
