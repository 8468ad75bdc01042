o=gpurun_out/r2w; mkdir -p $o
export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_v.so
for c in c5 c4; do
  CFGSIM_BIG_HIST=1 timeout 600 python tools/ab_bitwise.py $c $o/bw_${c}_hist.npz > $o/bw_${c}_hist.log 2>&1
  CFGSIM_BIG_HIST=0 timeout 600 python tools/ab_bitwise.py $c $o/bw_${c}_nohist.npz > $o/bw_${c}_nohist.log 2>&1
  echo "$c hist vs nohist: $(python tools/ab_bitwise.py cmp $o/bw_${c}_hist.npz $o/bw_${c}_nohist.npz)" >> $o/bitwise.txt
done
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_distributed.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
unset CFGSIM_LIBRARY
OUT=r2w VARS="s v s v" NOC2=1 bash tools/gpu_ab3.sh
