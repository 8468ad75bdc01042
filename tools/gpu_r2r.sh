o=gpurun_out/r2r; mkdir -p $o
export CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_prof2.so CFGSIM_PHASES=0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_big -c 1 -o $o/big16 python tools/phases.py c5 --graphs 600 > $o/ncu_big16.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_pair2 -c 1 -o $o/pair2 python tools/phases.py c2 > $o/ncu_pair2.log 2>&1
unset CFGSIM_LIBRARY CFGSIM_PHASES
timeout 600 python tools/e2e_breakdown.py > $o/e2e_breakdown.txt 2>&1
