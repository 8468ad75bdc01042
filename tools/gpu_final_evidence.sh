#!/bin/bash
# Round evidence: bench lines for every config, the C2 launch list and full
# ncu captures of the hot kernels.  Outputs under gpurun_out/final/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 300 python bench.py > $O/bench_c2.jsonl 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref_c2.jsonl 2>&1
timeout 600 python bench.py --config c3 --steps 1 --warmup 1 > $O/bench_c3.jsonl 2>&1
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --cpu-seconds 20 > $O/bench_c4.jsonl 2>&1
timeout 900 python bench.py --config c5 --graphs 3000 --steps 1 --warmup 1 --no-e2e > $O/bench_c5_3k.jsonl 2>&1
timeout 300 python bench.py --precision fp32 --no-cpu --no-e2e > $O/bench_c2_fp32.jsonl 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > $O/ncu_launches.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:isorank_pair2 -s 3 -c 1 -f -o $O/prof_pair2 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_pair2.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:isorank_seq4 -s 0 -c 1 -f -o $O/prof_seq4 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_seq4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:isorank_big -s 2 -c 1 -f -o $O/prof_big \
  python bench.py --config c4 --graphs 100 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_big.log 2>&1
echo done > $O/done
