#!/bin/bash
# GPU parity subset + bench lines of the given configs (reps interleaved)
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x -k "${KEXPR:-parity or fuzz or fullsize or robust or abi}" > $O/qc_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/qc_pytest.log)"
for rep in 1 2; do for c in ${CFGS:-c3 c2 c1}; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/qc.json 2>/dev/null
  echo "$c $(python -c "import json;d=json.load(open('$O/qc.json'));print(d['ms_per_step'], d['critical_path_ms'].get('no_big_gemm'))")"
done; done
