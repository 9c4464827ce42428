for r in 0 0.1 0.25 0.5 1.0; do
  BD_SUPER_RELAX=$r python tools/cfg_run.py --workload cfg1 --steps 25 > gpurun_out/rx_$r.log 2>&1
done
BD_SUPER_RELAX=0.25 python -m pytest tests/test_gpu_trsv_variants.py -q -p no:cacheprovider -k exact > gpurun_out/rx_tests.log 2>&1
