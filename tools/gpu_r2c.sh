mkdir -p gpurun_out/r2c
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2c/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2c/pytest.txt
CFGSIM_PHASES=1 timeout 600 python tools/phases.py c2 > gpurun_out/r2c/phases_c2.txt 2>&1
timeout 600 python bench.py --no-cpu --steps 5 --warmup 3 > gpurun_out/r2c/bench_c2.jsonl 2> gpurun_out/r2c/bench_c2.err
