mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a/pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/r2a/bench_c2.jsonl 2> gpurun_out/r2a/bench_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/r2a/bench_ref.jsonl 2> gpurun_out/r2a/bench_ref.err
timeout 1200 python bench.py --config c3 --steps 2 --warmup 1 > gpurun_out/r2a/bench_c3.jsonl 2> gpurun_out/r2a/bench_c3.err
bash tools/sanitize.sh > gpurun_out/r2a/sanitize_summary.txt 2>&1
