# session-3 A/B: stage-2 item claimed one pair ahead; phase shares and launch list of the current build
o=gpurun_out/s3e; mkdir -p $o
i=0
for v in bc6 claim bc6 claim; do
  i=$((i+1))
  CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_$v.so timeout 300 python bench.py --no-cpu --no-parity --no-e2e --steps 5 --warmup 3 > $o/c2_${i}_$v.jsonl 2> $o/c2_${i}_$v.err
done
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_claim.so CFGSIM_PHASES=1 timeout 600 python tools/phases.py c2 > $o/phases_c2.txt 2>&1
CFGSIM_LIBRARY=paper_1707_02423_b200/variants/libcfgsim_claim.so timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $o/launches_c2.csv \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-parity > $o/ncu_launches.log 2>&1
echo done > $o/done
