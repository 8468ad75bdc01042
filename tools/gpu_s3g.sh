# session-3 A/B: stage-2 consumer keeps the column after the head in a register (order load off the advance's path)
o=gpurun_out/s3g; mkdir -p $o
i=0
for v in claim nc1 claim nc1; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_nc1.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_nc1.so CFGSIM_PHASES=1 timeout 600 python tools/phases.py c2 > $o/phases_c2.txt 2>&1
echo done > $o/done
