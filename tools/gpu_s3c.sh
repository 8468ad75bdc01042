# session-3 A/B: stage-2 mma tiles dealt cyclically, tiles past N skipped; e2e breakdown
o=gpurun_out/s3c; mkdir -p $o
i=0
for v in ord tile ord tile; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 300 python tools/e2e_breakdown.py > $o/e2e_breakdown.txt 2>&1
timeout 400 python bench.py --no-cpu > $o/bench_c2_e2e.jsonl 2> $o/bench_c2_e2e.err
echo done > $o/done
