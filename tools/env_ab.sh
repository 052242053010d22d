#!/bin/bash
# Generic A/B test of one environment switch (under gpurun):
#   bash tools/env_ab.sh VAR "v1 v2" [reps] [config] [extra bench args]
# For every value: the GEMM parity tests and tools/bench_gemm.py once, then
# `bench.py` (c3 by default) `reps` times, values interleaved.
VAR=$1; VALS=$2; REPS=${3:-2}; CFG=${4:-c3}; EXTRA=${5:-}
O=gpurun_out; mkdir -p $O
for v in $VALS; do
  env $VAR=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -k dgemm > $O/ab_${v}_pytest.log 2>&1
  echo "$VAR=$v dgemm pytest rc=$? $(tail -1 $O/ab_${v}_pytest.log)"
  env $VAR=$v timeout 600 python tools/bench_gemm.py 2>&1 | sed "s/^/$VAR=$v /"
done
for rep in $(seq $REPS); do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv $EXTRA \
      > $O/ab_${v}_bench_$rep.json 2> $O/ab_${v}_bench_$rep.err
  echo "$VAR=$v $CFG rep $rep: $(python -c "import json;d=json.load(open('$O/ab_${v}_bench_$rep.json'));r=d['roofline'];print(d['ms_per_step'],'ms', r['achieved'], {k: v['ms'] for k, v in r['by_class'].items() if v['ms']})")"
done; done
