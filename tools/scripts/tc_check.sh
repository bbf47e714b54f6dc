mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tcgen05" > gpurun_out/pytest_tc.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_tc.log
timeout 900 python tools/quick_perf.py gemmf32 > gpurun_out/qp_gemm32.log 2>&1; echo qp rc=$?
python -c "
import json
for l in open('gpurun_out/qp_gemm32.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['variant'], round(d['ms'],3), round(d['gflops_mm']))
"
