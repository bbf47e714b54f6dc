mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_swar.py -x -q > gpurun_out/pytest_swar.log 2>&1; echo pytest swar rc=$?
tail -15 gpurun_out/pytest_swar.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "eqcount" > gpurun_out/pytest_eq.log 2>&1; echo pytest eq rc=$?
tail -5 gpurun_out/pytest_eq.log
timeout 900 python tools/quick_perf.py eqcount > gpurun_out/qp_eq.log 2>&1; echo qp rc=$?
python -c "
import json
for l in open('gpurun_out/qp_eq.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['variant'], round(d['ms'],3), round(d['gflops_mm']))
"
