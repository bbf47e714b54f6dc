mkdir -p gpurun_out tools/bin
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/thetabench tools/thetabench.cu && timeout 120 tools/bin/thetabench > gpurun_out/thetabench2.txt 2>&1
cat gpurun_out/thetabench2.txt
timeout 600 python -m pytest tests/test_gpu_theta.py -x -q > gpurun_out/pytest_theta.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_theta.log
timeout 900 python tools/quick_perf.py discount > gpurun_out/qp_discount.log 2>&1; echo qp rc=$?
grep -h '"shape": \[8192' gpurun_out/qp_discount.log | grep theta | python -c "import sys,json; [print(json.loads(l)['variant'], round(json.loads(l)['ms'],2), round(json.loads(l)['gflops_mm'])) for l in sys.stdin]"
