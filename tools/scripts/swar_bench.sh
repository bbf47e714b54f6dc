mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_swar.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload cfg3_eqcount_i32 --steps 10 --warmup 3 > gpurun_out/bench_cfg3b.json 2> gpurun_out/bench_cfg3b.err; echo bench rc=$?
cat gpurun_out/bench_cfg3b.json
W=$(python -c "import json;print(json.load(open('gpurun_out/bench_cfg3b.json'))['config']['tile'])")
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_cfg3b.csv python bench.py --workload cfg3_eqcount_i32 --steps 2 --warmup 1 --no-cpu --no-e2e --tile $W > gpurun_out/ncu_cfg3b.log 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:BodySwarEq -s 0 -c 1 -o gpurun_out/swar_cfg3b python bench.py --workload cfg3_eqcount_i32 --steps 1 --warmup 1 --no-cpu --no-e2e --tile $W > gpurun_out/ncu_full_cfg3b.log 2>&1; echo ncu full rc=$?
