o=gpurun_out/r2z; mkdir -p $o
export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_w.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sanitize.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
for v in h2 w; do CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python tools/ab_bitwise.py c2 $o/bw_c2_$v.npz > /dev/null 2>&1; done
echo "c2 h2 vs w: $(python tools/ab_bitwise.py cmp $o/bw_c2_h2.npz $o/bw_c2_w.npz)" > $o/bitwise.txt
unset CFGSIM_LIBRARY
i=0
for v in h2 w h2 w; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/bench_c2_${i}_$v.jsonl 2> $o/bench_c2_${i}_$v.err
done
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_w.so CFGSIM_PHASES=1 timeout 900 python tools/phases.py c2 > $o/phases_c2.txt 2>&1
