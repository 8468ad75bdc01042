#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (N=1), launch list and one
# full ncu capture of the hot kernel.  Outputs under gpurun_out/.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
if [ "${NCU:-1}" = 1 ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:isorank_lowrank -s 60 -c 3 -f \
  -o gpurun_out/prof python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_full.log 2>&1
fi
echo done
