# session-3 A/B: 6 x 6 mma tile instance for N <= 48
o=gpurun_out/s3d; mkdir -p $o
i=0
for v in ord bc6 ord bc6; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
for v in ord bc6; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c3 --no-cpu --no-parity --no-e2e --steps 2 --warmup 1 > $o/c3_$v.jsonl 2> $o/c3_$v.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
echo done > $o/done
