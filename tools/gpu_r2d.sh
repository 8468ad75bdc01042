mkdir -p gpurun_out/r2d
CFGSIM_PHASES=1 timeout 600 python tools/phases.py c4 --graphs 60 > gpurun_out/r2d/phases_c4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_large.py -x -q > gpurun_out/r2d/pytest_large.txt 2>&1; echo "rc=$?" >> gpurun_out/r2d/pytest_large.txt
timeout 900 python bench.py --config c4 --graphs 300 --no-cpu --no-e2e --steps 1 --warmup 1 > gpurun_out/r2d/bench_c4_300.jsonl 2> gpurun_out/r2d/bench_c4.err
