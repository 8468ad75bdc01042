# A/B on c4 / c5-subset: OUT=<dir> VARS="a b a b" bash tools/gpu_ab2.sh
o=gpurun_out/${OUT:-ab2}; mkdir -p $o
i=0
for v in ${VARS:-"a b"}; do
  i=$((i+1))
  export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
  timeout 900 python bench.py --config c4 --graphs ${C4G:-300} --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 > $o/bench_c4_${i}_$v.jsonl 2> $o/bench_c4_${i}_$v.err
  timeout 900 python bench.py --config c5 --graphs ${C5G:-1000} --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 > $o/bench_c5_${i}_$v.jsonl 2> $o/bench_c5_${i}_$v.err
done
unset CFGSIM_LIBRARY
if [ -n "$PHASES" ]; then CFGSIM_PHASES=1 timeout 900 python tools/phases.py c5 --graphs 600 > $o/phases_c5.txt 2>&1; fi
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt; fi
