#!/bin/bash
# A/B bench lines: ab.sh <workload> "<ENV=.. ENV2=..>" ... ; prints value / ms / frac per variant.
W=${W:-cfg3}
for v in "$@"; do
  env $v python bench.py --workload $W --engine ${E:-auto} --steps ${STEPS:-2} --warmup ${WARM:-2} --no-e2e --no-cpu 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W', '$v', round(d['value'],2), 'Tel/s', round(d['ms_per_step'],2), 'ms', round(d['roofline']['frac'],3))" 2>&1 | tail -1
done
