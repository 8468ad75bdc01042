o=gpurun_out/r2u; mkdir -p $o
export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_t.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
for i in 1 2; do
  CFGSIM_P2_OCC4=0 timeout 600 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/bench_c2_${i}_occ3.jsonl 2> $o/bench_c2_${i}_occ3.err
  CFGSIM_P2_OCC4=1 timeout 600 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/bench_c2_${i}_occ4.jsonl 2> $o/bench_c2_${i}_occ4.err
done
CFGSIM_PHASES=1 timeout 900 python tools/phases.py c2 > $o/phases_c2.txt 2>&1
timeout 900 python bench.py --no-cpu --no-parity > $o/bench_c2_full.jsonl 2> $o/bench_c2_full.err
timeout 600 python tools/e2e_breakdown.py > $o/e2e_breakdown.txt 2>&1
