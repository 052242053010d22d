O=gpurun_out; mkdir -p $O
run() { env $1 timeout 600 python bench.py --config $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/ab3.json 2>/dev/null; echo "$1 $2 $(python -c "import json;d=json.load(open('$O/ab3.json'));print(d['ms_per_step'])")"; }
timeout 900 python -m pytest tests -m gpu -q -x -k "parity or fuzz or fullsize" 2>&1 | tail -1
for rep in 1 2; do
for c in c1 c2 c3; do
  run "RANDUTV_SVD_MERGE_TAIL=0 RANDUTV_SVD_CHUNK=8" $c
  run "RANDUTV_SVD_MERGE_TAIL=1 RANDUTV_SVD_CHUNK=8" $c
  run "RANDUTV_SVD_MERGE_TAIL=1 RANDUTV_SVD_CHUNK=0" $c
done; done
for ch in 2 3 4 6; do run "RANDUTV_SVD_CHUNK=$ch" c2; run "RANDUTV_SVD_CHUNK=$ch" c1; done
