#!/bin/bash
# A/B of the SVD tail scheduling (RANDUTV_SVD_TAIL = 0 sequential, 1 merged, 2 concurrent)
O=gpurun_out; mkdir -p $O
run() { env $1 timeout 600 python bench.py --config $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/abt.json 2>/dev/null; echo "$1 $2 $(python -c "import json;d=json.load(open('$O/abt.json'));print(d['ms_per_step'], d['critical_path_ms'].get('tail_after_last_big_gemm'))")"; }
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or fuzz or fullsize or robust" 2>&1 | tail -1
for rep in 1 2; do for c in c3 c2 c1 c4; do for t in 2 1 0; do run "RANDUTV_SVD_TAIL=$t" $c; done; done; done
