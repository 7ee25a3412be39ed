#!/bin/bash
# One GPU measurement pass (run under gpurun):  bash tools/gpu_bench.sh <tag> [full]
#   gpurun_out/<tag>_bench.json      bench.py line (+ per-kernel breakdown)
#   gpurun_out/<tag>_launches.csv    ncu launch list (gpu__time_duration, clock-control none)
#   gpurun_out/<tag>_prof.ncu-rep    ncu --set full of k_sparse_attn, k_score and k_select (only with "full")
TAG=${1:-run}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { cat gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python bench.py --breakdown > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?"; tail -c 3000 gpurun_out/${TAG}_bench.json; tail -5 gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --e2e-steps 1 \
  --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "ncu launches rc=$?"
if [ "$2" == "full" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_sparse_attn|k_score|k_select|k_merge" -s 128 -c 4 \
    -o gpurun_out/${TAG}_prof python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_full.log 2>&1
  echo "ncu full rc=$?"
fi
