# dev: bench.py under several triangular-solve kernels (short runs, no CPU baseline)
for k in ${KERNELS:-smem reg pipe}; do
  echo "== $k"
  BD_BTILE_KERNEL=$k python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['value'], d['config']['ms_per_pcg_iter'], {k: round(v['ms']/max(1,v['marks']),4) for k,v in d['profile_ms'].items()})"
done
