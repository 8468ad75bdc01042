o=gpurun_out/r2v; mkdir -p $o
for v in s u; do for c in c5 c4; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python tools/ab_bitwise.py $c $o/bw_${c}_$v.npz > /dev/null 2>&1
done; done
for c in c5 c4; do echo "$c s vs u: $(python tools/ab_bitwise.py cmp $o/bw_${c}_s.npz $o/bw_${c}_u.npz)" >> $o/bitwise.txt; done
OUT=r2v VARS="s u s u" NOC2=1 bash tools/gpu_ab3.sh
timeout 900 python bench.py --no-cpu --no-parity > $o/bench_c2_full.jsonl 2> $o/bench_c2_full.err
