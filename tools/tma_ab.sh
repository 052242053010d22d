#!/bin/bash
# A/B test of the GEMM staging: cp.async (RANDUTV_GEMM_TMA=0) vs TMA (=1).
O=gpurun_out; mkdir -p $O
for v in 1 0; do
  RANDUTV_GEMM_TMA=$v timeout 600 python -m pytest tests/test_gpu_parity.py -q -k dgemm > $O/tma${v}_pytest.log 2>&1; echo "tma=$v pytest rc=$?"; tail -2 $O/tma${v}_pytest.log
  RANDUTV_GEMM_TMA=$v timeout 600 python tools/bench_gemm.py > $O/tma${v}_gemm.log 2>&1; cat $O/tma${v}_gemm.log
done
RANDUTV_TMA_NO3D=1 RANDUTV_GEMM_TMA=1 timeout 600 python tools/bench_gemm.py 2>&1 | head -3 | sed 's/^/no3d: /'
for rep in 1 2; do for v in 1 0; do
  RANDUTV_GEMM_TMA=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv > $O/tma${v}_bench_$rep.json 2>$O/tma${v}_bench_$rep.err
  echo "tma=$v c3 $(python -c "import json;d=json.load(open('$O/tma${v}_bench_$rep.json'));print(d['ms_per_step'], d['roofline']['achieved'])")"
done; done
