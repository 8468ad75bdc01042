o=gpurun_out/r2q; mkdir -p $o
for v in o n q; do
  for c in c5 c4; do
    CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python tools/ab_bitwise.py $c $o/bw_${c}_$v.npz > /dev/null 2>&1
  done
done
for c in c5 c4; do for v in n q; do echo "$c o vs $v: $(python tools/ab_bitwise.py cmp $o/bw_${c}_o.npz $o/bw_${c}_$v.npz)" >> $o/bitwise.txt; done; done
OUT=r2q VARS="o n q o n q" NOC2=1 bash tools/gpu_ab3.sh
timeout 1500 python tools/c5_full.py --ranks 7 --out $o/c5_rank7.json > $o/c5_rank7.log 2>&1
