#!/bin/bash
# One gpurun call collecting a round's evidence: GPU tests, the default bench
# line, the --dist bench line (NCCL, 1 rank), the reference arm, GEMM-vs-cuBLAS,
# the ncu launch list of the bench command itself (--steps 1 --warmup 3, no
# extras: cold-cache, serialised per-launch times -> shares, not absolutes),
# the library's live timeline, one full ncu capture of the dominant GEMM shapes
# and of the DSMEM Cholesky.  Usage (under gpurun):  bash tools/gpu_evidence.sh TAG
TAG=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 $O/${TAG}_pytest.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
tail -c 3000 $O/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/${TAG}_bench_reference.json 2>&1; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29513 bench.py --gpus 1 --dist --no-cpu-baseline 2> $O/${TAG}_bench_dist_n1.err | tail -1 \
    > $O/${TAG}_bench_dist_n1.json; echo "dist bench rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-utv > $O/${TAG}_bench_$c.json 2>&1
done
timeout 600 python tools/bench_gemm.py > $O/${TAG}_gemm.log 2>&1; tail -5 $O/${TAG}_gemm.log
TIMELINE_OUT=$O/${TAG}_timeline.json timeout 600 python tools/timeline.py c3 > $O/${TAG}_timeline.txt 2>&1
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-utv --no-cpu-baseline"
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${TAG}_launches.csv $B > $O/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/prof_gemm.py > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dgemm -s 9 -c 3 \
    -o $O/${TAG}_gemm python tools/prof_gemm.py > $O/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
[ -x tools/chol_bench ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_inv_dsm \
    -s 1 -c 1 -o $O/${TAG}_chol ./tools/chol_bench 256 1e3 > $O/${TAG}_ncu_chol.log 2>&1; echo "ncu chol rc=$?"
timeout 600 python tools/gemm_steps.py > $O/${TAG}_gemm_steps.txt 2>&1; echo "gemm steps rc=$?"
RANDUTV_EXP_NO_SWEEPS=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-utv \
    > $O/${TAG}_bench_nosweeps.json 2>/dev/null; echo "no-sweeps timing rc=$?"
cuobjdump -sass paper_1703_00998_b200/_randutv.so > /tmp/sass.txt 2>/dev/null && \
  for op in DMMA LDGSTS UTMALDG UTMASTG DFMA HMMA UTCHMMA UTCQMMA; do echo "$op $(grep -c "$op" /tmp/sass.txt)"; done \
  > $O/${TAG}_sass_counts.txt
