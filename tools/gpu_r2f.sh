mkdir -p gpurun_out/r2f
export CFGSIM_PHASES=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_pair2 -c 1 -o gpurun_out/r2f/pair2 python tools/phases.py c2 > gpurun_out/r2f/ncu_pair2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_big -c 1 -o gpurun_out/r2f/big python tools/phases.py c4 --graphs 40 > gpurun_out/r2f/ncu_big.log 2>&1
