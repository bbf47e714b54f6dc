set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_theta.py -x -q > gpurun_out/pytest_theta.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_theta.log
timeout 900 python tools/quick_perf.py discount > gpurun_out/qp_discount.log 2>&1; echo qp rc=$?
grep -h '"shape": \[8192' gpurun_out/qp_discount.log | python -c "import sys,json; [print(json.loads(l)['variant'], round(json.loads(l)['ms'],2), round(json.loads(l)['gflops_mm'])) for l in sys.stdin]"
tail -3 gpurun_out/qp_discount.log
