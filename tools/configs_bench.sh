#!/bin/bash
# Main-line bench of the batched / long configs (run under gpurun): bash tools/configs_bench.sh <tag> [configs...]
TAG=${1:-cfg}; shift
CFGS=${@:-c3 c5 c4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
for c in $CFGS; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline --vc-rho "${VC:-}" \
    --q-len-leg ${QL:-0} --lowrank-gen-leg 0 > gpurun_out/${TAG}_${c}.json 2> gpurun_out/${TAG}_${c}.err
  python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_${c}.json").read().strip().splitlines()[-1])
print("$c", round(d["value"], 1), "ms", round(d["ms_per_step"], 3), "frac", round(d["roofline"]["frac"], 3),
      "step_frac", round(d["roofline"].get("step_frac_of_roofline", 0), 3), "vc", d.get("value_cache", {}).get("value"))
PY
done
