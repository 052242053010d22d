#!/bin/bash
# split-K reduction A/B: mode 0 (HBM partials) vs mode 1/2 at output-size thresholds
O=gpurun_out; mkdir -p $O
for rep in 1 2; do for c in c2 c1 c3; do for v in "0 0" "1 0" "1 16384" "1 131072" "2 16384"; do
  set -- $v
  RANDUTV_GEMM_CLUSTER=$1 RANDUTV_GEMM_CLUSTER_MIN=$2 timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/csk.json 2>/dev/null
  echo "$c mode=$1 min=$2 $(python -c "import json;d=json.loads(open('$O/csk.json').read().strip().splitlines()[-1]);print(d['ms_per_step'])")"
done; done; done
