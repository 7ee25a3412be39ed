#!/bin/bash
# A/B of an environment switch on the c2 main line (run under gpurun): bash tools/ab.sh VAR reps
VAR=$1; REPS=${2:-3}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in $(seq $REPS); do for v in 0 1; do
  env $VAR=$v timeout 300 python bench.py --steps 300 --warmup 5 --e2e-steps 3 --no-cpu-baseline --vc-rho "" --q-len-leg 0 \
    --lowrank-gen-leg 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$VAR=$v', round(d['value'],1), round(d['ms_per_step'],4))"
done; done
