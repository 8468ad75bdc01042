# session-3 A/B: large-N greedy prefetches each row's coming sorted entries to L2
o=gpurun_out/s3k; mkdir -p $o
for v in claim l2pf l2pf48 claim l2pf l2pf48; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c4 --graphs 300 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 >> $o/c4_$v.jsonl 2>> $o/c4_$v.err
done
for v in claim l2pf l2pf48; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c5 --graphs 1000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 > $o/c5_$v.jsonl 2> $o/c5_$v.err
done
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_l2pf.so timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
echo done > $o/done
