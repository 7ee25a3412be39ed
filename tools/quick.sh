#!/bin/bash
# Quick GPU iteration (run under gpurun):  bash tools/quick.sh <tag> [pytest-args...]
#   build; the GPU parity tests (or the given subset); a short c2 bench without the widened legs;
#   a 6-layer steady-state trace.  Outputs under gpurun_out/<tag>_*.
TAG=${1:-quick}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail -30 gpurun_out/${TAG}_build.log; exit 1; }
if [ "$1" != "none" ]; then
  timeout 900 python -m pytest -m gpu -x -q -p no:cacheprovider ${@:-tests} > gpurun_out/${TAG}_pytest.log 2>&1
  echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest.log
fi
timeout 600 python bench.py --steps 200 --warmup 5 --e2e-steps 10 --no-cpu-baseline --vc-rho 0.95 --q-len-leg 0 \
  --lowrank-gen-leg 0 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python - <<EOF
import json
d = json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "ms", round(d["ms_per_step"], 4), "frac", round(d["roofline"]["frac"], 3))
vc = d.get("value_cache") or []
for leg in (vc if isinstance(vc, list) else [vc]):
    print("  vc C/k", leg.get("capacity_over_k"), "value", round(leg.get("value", 0), 1), "alpha", round(leg.get("alpha", 0), 3),
          "frac", round(leg.get("step_frac_of_host_roofline", 0), 3), leg.get("error", ""))
EOF
timeout 300 python tools/trace_run.py --slots 6 > gpurun_out/${TAG}_trace_c2.txt 2>&1
head -9 gpurun_out/${TAG}_trace_c2.txt
