#!/bin/bash
# Bench lines for every config (GPU box).  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.log 2>&1
timeout 1200 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --cpu-seconds 20 > gpurun_out/bench_c4.log 2>&1
timeout 1200 python bench.py --config c3 --graphs 20000 --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_c3_20k.log 2>&1
timeout 1200 python bench.py --config c5 --graphs 3000 --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_c5_3k.log 2>&1
echo done
