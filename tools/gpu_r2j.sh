mkdir -p gpurun_out/r2j
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2j/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/r2j/pytest_gpu.txt
timeout 900 python bench.py > gpurun_out/r2j/bench_c2.jsonl 2> gpurun_out/r2j/bench_c2.err
timeout 2400 python tools/calibrate_split.py --out gpurun_out/r2j/cost.json > gpurun_out/r2j/calib.log 2>&1
