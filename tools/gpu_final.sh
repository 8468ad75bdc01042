# Round-end evidence: GPU tests, bench lines for every config, the reference
# arm, C5 at full size as 8 ranks, ncu launch list + full captures.
o=gpurun_out/final; mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1; echo "rc=$?" >> $o/pytest_gpu.txt
timeout 900 python bench.py > $o/bench_c2.jsonl 2> $o/bench_c2.err
timeout 900 python bench.py --precision fp32 --no-cpu > $o/bench_c2_fp32.jsonl 2> $o/bench_c2_fp32.err
timeout 900 python bench.py --impl reference > $o/bench_ref_c2.jsonl 2> $o/bench_ref_c2.err
timeout 1500 python bench.py --config c3 --steps 2 --warmup 3 > $o/bench_c3.jsonl 2> $o/bench_c3.err
timeout 1500 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > $o/bench_c4.jsonl 2> $o/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $o/c2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-parity > $o/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_pair2 -c 1 -o $o/pair2 python tools/phases.py c2 > $o/ncu_pair2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:isorank_big -c 1 -o $o/big16 python tools/phases.py c5 --graphs 600 > $o/ncu_big16.log 2>&1
CFGSIM_PHASES=1 timeout 900 python tools/phases.py c5 --graphs 600 > $o/phases_c5.txt 2>&1
CFGSIM_PHASES=1 timeout 900 python tools/phases.py c2 > $o/phases_c2.txt 2>&1
timeout 4000 python tools/c5_full.py --out $o/c5_full.json > $o/c5_full.log 2>&1
