# session-3: ncu full capture of the first large-N launch of a C5-distribution corpus (same command as profiles/r02_c5_big16_ncu_full.txt)
o=gpurun_out/s3o; mkdir -p $o
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:isorank_big -c 1 -f -o $o/big16 python tools/phases.py c5 --graphs 600 > $o/ncu_big16.log 2>&1
echo done > $o/done
