# dev A/B of an env knob in the full bench on one box: bash tools/_ab/bench_ab.sh KNOB
K=${1:-BD_PREFILL}
for r in 1 2; do for v in 0 1; do
env $K=$v python bench.py --no-cpu > gpurun_out/ab_$v.json 2>/dev/null
python - <<EOF
import json
d=json.loads(open("gpurun_out/ab_$v.json").read().strip().splitlines()[-1])
print("$K=$v", d["value"], d["e2e"]["value"], d["config"]["ms_per_pcg_iter"], d["config"]["pcg_iters_per_step"], {k: round(x["ms"],1) for k,x in d["profile_ms"].items()})
EOF
done; done
