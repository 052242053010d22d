#!/bin/bash
# One gpurun call: GPU tests, the default bench line, the --dist bench line (NCCL, 1 rank), GEMM-vs-cuBLAS table,
# the ncu launch list of one factorization (tools/prof_step.py: 1 warm-up + 1
# profiled step; the summary keeps the last step's launches) and one full ncu
# capture of the three dominant GEMM shapes.  Usage (under gpurun):
#   bash tools/gpu_evidence.sh TAG
TAG=${1:-r01}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/${TAG}_pytest.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
cat $O/${TAG}_bench.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 1 --dist --no-cpu-baseline 2> $O/${TAG}_bench_dist_n1.err | tail -1 \
    > $O/${TAG}_bench_dist_n1.json; echo "dist bench rc=$?"
timeout 600 python tools/bench_gemm.py > $O/${TAG}_gemm.log 2>&1; cat $O/${TAG}_gemm.log
P="python tools/prof_step.py c3 1"
$P > $O/${TAG}_prof_plain.log 2>&1 && cat $O/${TAG}_prof_plain.log && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_launches.csv $P > $O/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
N=$(grep -o 'launches_per_step=[0-9]*' $O/${TAG}_prof_plain.log | cut -d= -f2)
python tools/launch_summary.py $O/${TAG}_launches.csv ${N:-0} > $O/${TAG}_launch_summary.txt; head -30 $O/${TAG}_launch_summary.txt
python tools/prof_gemm.py > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 9 -c 3 \
    -o $O/${TAG}_gemm python tools/prof_gemm.py > $O/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
