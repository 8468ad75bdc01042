# A/B of prebuilt library variants (tools/build_variant.sh):
#   OUT=<dir> VARS="a b a b" [TESTS=1] [NOC4=1] [C4G=300] bash tools/gpu_ab.sh
# (a variant may repeat: runs are numbered in order, to expose box noise)
o=gpurun_out/${OUT:-ab}; mkdir -p $o
V=${VARS:-"a base"}
if [ -n "$TESTS" ]; then
  for v in $(echo $V | tr ' ' '\n' | sort -u); do
    export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
    timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q > $o/pytest_$v.txt 2>&1; echo "rc=$?" >> $o/pytest_$v.txt
  done
fi
i=0
for v in $V; do
  i=$((i+1))
  export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
  timeout 600 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/bench_c2_${i}_$v.jsonl 2> $o/bench_c2_${i}_$v.err
  if [ -z "$NOC4" ]; then
    timeout 900 python bench.py --config c4 --graphs ${C4G:-300} --no-cpu --no-e2e --no-parity --steps 2 --warmup 1 > $o/bench_c4_${i}_$v.jsonl 2> $o/bench_c4_${i}_$v.err
  fi
done
unset CFGSIM_LIBRARY
