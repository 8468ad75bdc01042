# session-3 A/B: consumer heads as row-encoded keys (one 32-bit shuffle per round); e2e host-stall diagnostics
o=gpurun_out/s3h; mkdir -p $o
i=0
for v in claim renc claim renc; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_renc.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 300 python tools/e2e_stalls.py > $o/stalls_default.txt 2>&1
CFGSIM_HOST_THREADS=2 OMP_NUM_THREADS=1 timeout 300 python tools/e2e_stalls.py > $o/stalls_t2.txt 2>&1
timeout 300 python tools/e2e_stalls.py > $o/stalls_default2.txt 2>&1
echo done > $o/done
