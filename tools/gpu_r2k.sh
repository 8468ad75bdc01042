mkdir -p gpurun_out/r2k
export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_prof1.so CFGSIM_PHASES=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_big -c 1 -o gpurun_out/r2k/big python tools/phases.py c4 --graphs 40 > gpurun_out/r2k/ncu_big.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_pair2 -c 1 -o gpurun_out/r2k/pair2 python tools/phases.py c2 > gpurun_out/r2k/ncu_pair2.log 2>&1
unset CFGSIM_LIBRARY
timeout 1200 python tools/calibrate_split.py --out gpurun_out/r2k/cost.json > gpurun_out/r2k/calib.log 2>&1
