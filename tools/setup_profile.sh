# dev: host setup stages of the IC(0) inners at the cfg4 192^3 sweep point and cfg2
BD_DEBUG=1 python tools/cfg_run.py --workload cfg4 --cells 192 --steps 1 2>&1 | grep -E "setup|precond"
BD_DEBUG=1 python tools/cfg_run.py --workload cfg2 --steps 1 2>&1 | grep -E "setup|precond"
