#!/bin/bash
# A/B of the split-K reduction (RANDUTV_GEMM_CLUSTER=0 HBM partials + reduce,
# 1 cluster epilogue, 2 cluster-costed plans): GEMM parity, then bench ms per
# factorization of c3 / c2 / c1, modes interleaved, two rounds.
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dgemm" > $O/csk_pytest.log 2>&1; echo "gemm pytest rc=$? $(tail -1 $O/csk_pytest.log)"
for rep in 1 2; do for c in ${CFGS:-c3 c2 c1}; do for mode in ${MODES:-0 1 2}; do
  RANDUTV_GEMM_CLUSTER=$mode timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/csk.json 2>/dev/null
  echo "$c mode=$mode $(python -c "import json;d=json.loads(open('$O/csk.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['critical_path_ms'].get('no_big_gemm'), d['roofline']['achieved'])")"
done; done; done
