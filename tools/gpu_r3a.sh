o=gpurun_out/r3a; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distributed.py tests/test_gpu_sanitize.py -q -x > $o/pytest.txt 2>&1; echo "rc=$?" >> $o/pytest.txt
timeout 1500 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu > $o/bench_c3.jsonl 2> $o/bench_c3.err
