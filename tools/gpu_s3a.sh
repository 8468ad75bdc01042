# session-3 A/B: stage-2 row-order network without per-exchange direction selects
o=gpurun_out/s3a; mkdir -p $o
i=0
for v in base sortfix base sortfix; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -m gpu -x -q > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:isorank_pair2 -s 3 -c 1 -f -o $o/prof_pair2 \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity > $o/ncu_pair2.log 2>&1
ncu -i $o/prof_pair2.ncu-rep --page source --csv --print-source sass > $o/pair2_sass.csv 2>&1
ncu -i $o/prof_pair2.ncu-rep --page raw --csv > $o/pair2_raw.csv 2>&1
echo done > $o/done
