#!/bin/bash
# Full GPU suite at the default split-K mode, then c3/c2/c1 at modes 0 / 2 (3 rounds, interleaved)
O=gpurun_out; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/csk2_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 $O/csk2_pytest.log)"
grep -E "FAILED|Error" $O/csk2_pytest.log | head -10
for rep in 1 2 3; do for c in c3 c2 c1; do for mode in 0 2; do
  RANDUTV_GEMM_CLUSTER=$mode timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/csk.json 2>/dev/null
  echo "$c mode=$mode $(python -c "import json;d=json.loads(open('$O/csk.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['critical_path_ms'].get('no_big_gemm'), d['roofline']['achieved'])")"
done; done; done
