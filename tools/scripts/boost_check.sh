mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "boost" > gpurun_out/pytest_boost.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_boost.log
timeout 900 python tools/quick_perf.py boostf64 > gpurun_out/qp_boost.log 2>&1; echo qp rc=$?
python -c "
import json
for l in open('gpurun_out/qp_boost.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['variant'], round(d['ms'],3), round(d['gflops_mm']))
"
