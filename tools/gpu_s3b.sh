# session-3 A/B: packed row-order stores + lazy tie check (stage 2), fixed-direction large-N sort
o=gpurun_out/s3b; mkdir -p $o
i=0
for v in sortfix ord sortfix ord; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
for v in sortfix ord; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c4 --graphs 300 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 > $o/c4_$v.jsonl 2> $o/c4_$v.err
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --config c5 --graphs 1000 --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 > $o/c5_$v.jsonl 2> $o/c5_$v.err
done
timeout 1200 python -m pytest tests -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
echo done > $o/done
