o=gpurun_out/r2n; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sanitize.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 20 python tools/sanitize_run.py c2 --graphs 64 > $o/${tool}_c2.log 2>&1
  echo "$tool c2 rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|bitwise' $o/${tool}_c2.log | tr '\n' ' ')" >> $o/sanitize.txt
done
i=0
for v in j k l j k l; do
  i=$((i+1))
  export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
  timeout 600 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/bench_c2_${i}_$v.jsonl 2> $o/bench_c2_${i}_$v.err
done
unset CFGSIM_LIBRARY
CFGSIM_PHASES=1 timeout 900 python tools/phases.py c2 > $o/phases_c2.txt 2>&1
timeout 900 python bench.py > $o/bench_full.jsonl 2> $o/bench_full.err
