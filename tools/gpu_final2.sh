o=gpurun_out/final2; mkdir -p $o
{ nproc; python -c "import os; print(len(os.sched_getaffinity(0)), os.cpu_count())"; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/cpu/cpu.cfs_quota_us 2>/dev/null; uptime; } > $o/host.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_parity.py -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 900 python bench.py > $o/bench_c2.jsonl 2> $o/bench_c2.err
timeout 900 python tools/e2e_breakdown.py > $o/e2e_breakdown.txt 2>&1
timeout 1500 python bench.py --config c3 --steps 2 --warmup 3 --no-cpu > $o/bench_c3.jsonl 2> $o/bench_c3.err
timeout 4000 python tools/c5_full.py --out $o/c5_full.json > $o/c5_full.log 2>&1
