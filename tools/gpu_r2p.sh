o=gpurun_out/r2p; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 900 python bench.py > $o/bench_c2.jsonl 2> $o/bench_c2.err
timeout 900 python bench.py --impl reference > $o/bench_ref.jsonl 2> $o/bench_ref.err
timeout 3000 python tools/c5_full.py --out $o/c5_full.json > $o/c5_full.log 2>&1
