# session-3 A/B: large-N L2 prefetch modes (0: N <= 512 every advance; 1: once per 16 entries, all N; 2: 0 + column lines at N > 512)
o=gpurun_out/s3m; mkdir -p $o
for v in pfm0 pfm1 pfm2 pfm0 pfm1 pfm2; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c4 --graphs 300 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 >> $o/c4_$v.jsonl 2>> $o/c4_$v.err
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c5 --graphs 1000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 >> $o/c5_$v.jsonl 2>> $o/c5_$v.err
done
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_pfm1.so timeout 600 python -m pytest tests/test_gpu_large.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
echo done > $o/done
