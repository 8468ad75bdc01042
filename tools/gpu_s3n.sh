# session-3 A/B: large-N L2 prefetch distance (entries past the register window) at N <= 512
o=gpurun_out/s3n; mkdir -p $o
for v in ah16 ah8 ah32 ah16 ah8 ah32; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c5 --graphs 1000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 >> $o/c5_$v.jsonl 2>> $o/c5_$v.err
done
echo done > $o/done
