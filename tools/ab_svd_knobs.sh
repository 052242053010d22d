#!/bin/bash
# A/B of the SVD scheduling knobs on the latency-bound configs (bench ms per factorization)
for v in "" "RANDUTV_EXP_NO_SWEEPS=1" "RANDUTV_SVD_CHUNK=1" "RANDUTV_SVD_CHUNK=3" "RANDUTV_SVD_CHUNK=5" "RANDUTV_SVD_TAIL=1" "RANDUTV_SVD_TAIL=0"; do
  for c in c1 c2; do
    r=$(env $v timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-utv 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['ms_per_step'])")
    echo "$v $c $r"
  done
done
