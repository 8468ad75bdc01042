# Session-3 round evidence: bench lines for every config, C2 launch list, ncu full of the stage-2 kernel, phases
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/final3
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
timeout 400 python bench.py > $O/bench_c2.jsonl 2> $O/bench_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref_c2.jsonl 2> $O/bench_ref_c2.err
timeout 300 python bench.py --precision fp32 --no-cpu --no-e2e > $O/bench_c2_fp32.jsonl 2> $O/bench_c2_fp32.err
timeout 900 python bench.py --config c3 --steps 1 --warmup 1 > $O/bench_c3.jsonl 2> $O/bench_c3.err
timeout 900 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --cpu-seconds 20 > $O/bench_c4.jsonl 2> $O/bench_c4.err
CFGSIM_PHASES=1 timeout 600 python tools/phases.py c2 > $O/phases_c2.txt 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_c2.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $O/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:isorank_pair2 -s 3 -c 1 -f -o $O/prof_pair2 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > $O/ncu_pair2.log 2>&1
ncu -i $O/prof_pair2.ncu-rep --page raw --csv > $O/pair2_raw.csv 2>&1
echo done > $O/done
