#!/bin/bash
# Quick GPU iteration: GPU tests (no -x, all failures listed) + a short bench line.
# Usage (under gpurun): bash tools/gpu_quick.sh TAG [pytest -k expr]
TAG=${1:-q}
O=gpurun_out
mkdir -p $O
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 900 python -m pytest tests -m gpu -q $K > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 $O/${TAG}_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
cat $O/${TAG}_bench.json; tail -5 $O/${TAG}_bench.err
