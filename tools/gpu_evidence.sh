#!/bin/bash
# One gpurun call: GPU tests, the default bench line, GEMM-vs-cuBLAS table,
# the ncu launch list of one timed bench step and one full ncu capture of the
# top GEMM kernel.  Usage (under gpurun): bash tools/gpu_evidence.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/${TAG}_pytest.log
python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
cat $O/${TAG}_bench.json
python tools/bench_gemm.py > $O/${TAG}_gemm.log 2>&1; cat $O/${TAG}_gemm.log
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-utv"
$B > $O/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s ${SKIP:-31400} -c ${CNT:-11000} --csv \
    --log-file $O/${TAG}_launches.csv $B > $O/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py $O/${TAG}_launches.csv | head -30
P="python tools/prof_step.py c3 1"
$P > $O/${TAG}_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'dgemm_kernel<128' -s 0 -c 3 \
    -o $O/${TAG}_gemm $P > $O/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
