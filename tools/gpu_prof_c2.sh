#!/bin/bash
# Launch list + full ncu captures of the C2 bench kernels (stage-1 sequences,
# stage-2 pair kernel).  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:isorank_pair2 -s 40 -c 2 -f \
  -o gpurun_out/prof_pair2 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_p2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:isorank_seq -s 1 -c 1 -f \
  -o gpurun_out/prof_seq python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_seq.log 2>&1
echo done
