# C5 at full size with the session-3 build (8 rank ranges on one GPU) + host steal-time record during an e2e run
o=gpurun_out/s3j; mkdir -p $o
bash tools/steal.sh > $o/procstat.txt 2>&1 &
SP=$!
timeout 300 python tools/e2e_stalls2.py > $o/stalls2.txt 2>&1
kill $SP
timeout 2700 python tools/c5_full.py --out $o/c5_full.json > $o/c5_full.txt 2>&1
echo done > $o/done
