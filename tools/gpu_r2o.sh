o=gpurun_out/r2o; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 900 python bench.py > $o/bench_full.jsonl 2> $o/bench_full.err
CFGSIM_PIPELINE=0 timeout 900 python bench.py --no-cpu --no-parity > $o/bench_nopipe.jsonl 2> $o/bench_nopipe.err
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 20 python tools/sanitize_run.py c2 --graphs 64 > $o/${tool}_c2.log 2>&1
  echo "$tool c2 rc=$? :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|bitwise' $o/${tool}_c2.log | tr '\n' ' ')" >> $o/sanitize.txt
done
