o=gpurun_out/r2x; mkdir -p $o
export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_v.so
for spec in "1500 300 330" "1500 420 450" "1200 180 200"; do
  for h in 0 1 0 1; do CFGSIM_BIG_HIST=$h timeout 900 python tools/hist_ab.py $spec >> $o/hist_$h.txt 2>&1; done
done
unset CFGSIM_LIBRARY
OUT=r2x VARS="s v s v" NOC2=1 bash tools/gpu_ab3.sh
