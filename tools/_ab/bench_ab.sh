# dev A/B of an env knob in the full bench on one box: bash tools/_ab/bench_ab.sh KNOB v1 v2 [v3]
K=${1:-BD_PREFILL}
shift
for r in 1 2 3; do for v in "$@"; do
env $K=$v python bench.py --no-cpu --steps 20 > gpurun_out/ab_$v.json 2>/dev/null
python - <<EOF
import json
d=json.loads(open("gpurun_out/ab_$v.json").read().strip().splitlines()[-1])
print("$K=$v", d["value"], d["e2e"]["value"], d["config"]["ms_per_pcg_iter"])
EOF
done; done
