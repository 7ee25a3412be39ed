#!/bin/bash
# One gpurun call that produces a round's evidence:  bash tools/verify.sh <tag> [quick]
#   <tag>_pytest.log      the whole GPU suite (pytest -m gpu)
#   <tag>_smoke.log       __graft_entry__.smoke()
#   <tag>_bench.json      default bench line (c2 headline + legs)
#   <tag>_launches.csv    ncu launch list of a short c2 bench (gpu__time_duration, clock-control none)
#   <tag>_prof.ncu-rep    ncu --set full of the decode kernels (k_sparse_attn / score / select / merge)
#   <tag>_c3/c4/c5.json   main-line bench of the batched / long configs (skipped with "quick")
TAG=${1:-verify}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail -30 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1500 python -m pytest -m gpu -q -p no:cacheprovider tests > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -4 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"
python - <<EOF
import json
d = json.loads(open("gpurun_out/${TAG}_bench.json").read().strip().splitlines()[-1])
r = d["roofline"]
print("c2", round(d["value"], 1), "tok/s", round(d["ms_per_step"], 4), "ms e2e", round(d["e2e"]["value"], 1),
      "frac", round(r["frac"], 3), "step_frac", round(r.get("step_frac_of_roofline", 0), 3), "clocks", d.get("clocks"))
vc = d.get("value_cache") or []
for leg in (vc if isinstance(vc, list) else [vc]):
    print("  vc C/k", leg.get("capacity_over_k"), "value", round(leg.get("value", 0), 1), "alpha",
          round(leg.get("alpha", 0), 3), "frac", round(leg.get("step_frac_of_host_roofline", 0), 3), leg.get("error", ""))
EOF
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sparse_attn|k_score|k_select|k_merge" \
  -s 128 -c 4 -o gpurun_out/${TAG}_prof python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
if [ "$2" != "quick" ]; then
  bash tools/configs_bench.sh ${TAG} c3 c5 c4
fi
