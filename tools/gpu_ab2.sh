#!/bin/bash
# A/B of one env switch on the factorization only: GPU parity subset + c3 (and
# optionally c2/c1) bench lines, values interleaved.
#   bash tools/gpu_ab2.sh VAR "v1 v2" reps "configs" [pytest -k expr]
VAR=$1; VALS=$2; REPS=${3:-2}; CFGS=${4:-c3}; KEXPR=${5:-}
O=gpurun_out; mkdir -p $O
if [ -n "$KEXPR" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x -k "$KEXPR" > $O/ab2_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/ab2_pytest.log)"
fi
for rep in $(seq $REPS); do for c in $CFGS; do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv \
      > $O/ab2_${c}_${v}_$rep.json 2> $O/ab2_${c}_${v}_$rep.err
  echo "$VAR=$v $c rep $rep: $(python -c "import json;d=json.load(open('$O/ab2_${c}_${v}_$rep.json'));r=d['roofline'];cp=d.get('critical_path_ms',{});print(d['ms_per_step'],'ms exposed',cp.get('qr_chain_main_exposed'))" 2>&1 | tail -1)"
done; done; done
