o=gpurun_out/r3b; mkdir -p $o
for v in h3 x; do for c in c5 c4; do
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 600 python tools/ab_bitwise.py $c $o/bw_${c}_$v.npz > /dev/null 2>&1
done; done
for c in c5 c4; do echo "$c h3 vs x: $(python tools/ab_bitwise.py cmp $o/bw_${c}_h3.npz $o/bw_${c}_x.npz)" >> $o/bitwise.txt; done
OUT=r3b VARS="h3 x h3 x" NOC2=1 bash tools/gpu_ab3.sh
for h in h3 x; do CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$h.so timeout 900 python tools/hist_ab.py 1500 300 330 >> $o/hist_$h.txt 2>&1; done
