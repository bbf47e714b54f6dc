set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out tools/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/thetabench tools/thetabench.cu && timeout 120 tools/bin/thetabench > gpurun_out/thetabench.txt 2>&1
cat gpurun_out/thetabench.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu.log
