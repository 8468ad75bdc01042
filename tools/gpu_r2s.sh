o=gpurun_out/r2s; mkdir -p $o
for v in q r; do for c in c5 c4; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python tools/ab_bitwise.py $c $o/bw_${c}_$v.npz > /dev/null 2>&1
done; done
for c in c5 c4; do echo "$c q vs r: $(python tools/ab_bitwise.py cmp $o/bw_${c}_q.npz $o/bw_${c}_r.npz)" >> $o/bitwise.txt; done
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
OUT=r2s VARS="q r q r" NOC2=1 bash tools/gpu_ab3.sh
CFGSIM_PHASES=1 timeout 900 python tools/phases.py c5 --graphs 600 > $o/phases_c5.txt 2>&1
timeout 600 python tools/e2e_breakdown.py > $o/e2e_breakdown.txt 2>&1
timeout 900 python bench.py --no-cpu --no-parity > $o/bench_c2.jsonl 2> $o/bench_c2.err
