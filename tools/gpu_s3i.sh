o=gpurun_out/s3i; mkdir -p $o
timeout 300 python tools/e2e_stalls2.py > $o/stalls2.txt 2>&1
CUDA_DEVICE_MAX_CONNECTIONS=1 timeout 300 python tools/e2e_stalls2.py > $o/stalls2_b.txt 2>&1
echo done > $o/done
