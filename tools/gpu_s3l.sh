# session-3 A/B: L2 prefetch in the large-N greedy only for N <= 512
o=gpurun_out/s3l; mkdir -p $o
for v in claim l2pf16 claim l2pf16; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c5 --graphs 1000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 >> $o/c5_$v.jsonl 2>> $o/c5_$v.err
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c4 --graphs 300 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 >> $o/c4_$v.jsonl 2>> $o/c4_$v.err
done
echo done > $o/done
