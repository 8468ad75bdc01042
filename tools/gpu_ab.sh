# A/B of prebuilt library variants (tools/build_variant.sh):  OUT=<dir> VARS="a b c" bash tools/gpu_ab.sh
o=gpurun_out/${OUT:-ab}; mkdir -p $o
V=${VARS:-"a base"}
for v in $V; do
  export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_large.py -x -q > $o/pytest_$v.txt 2>&1; echo "rc=$?" >> $o/pytest_$v.txt
done
for v in $V; do
  export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
  timeout 600 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/bench_c2_$v.jsonl 2> $o/bench_c2_$v.err
done
if [ -z "$NOC4" ]; then
for v in $V; do
  export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so
  timeout 900 python bench.py --config c4 --graphs ${C4G:-300} --no-cpu --no-e2e --no-parity --steps 1 --warmup 1 > $o/bench_c4_$v.jsonl 2> $o/bench_c4_$v.err
done
fi
unset CFGSIM_LIBRARY
