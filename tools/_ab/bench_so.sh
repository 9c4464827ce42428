# dev A/B of two library builds in the full bench on one box (tools/_ab/base.bin, new.bin)
for r in 1 2 3; do for v in base new; do
cp tools/_ab/$v.bin paper_1711_08708_b200/libbidomain_b200.so
python bench.py --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['config']['ms_per_pcg_iter'])"
done; done
