mkdir -p gpurun_out/bench_lines
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for w in cfg1_boost_f32 cfg1_boost_f64 cfg3_sqdiff_f32 cfg0_discount_f64 cfg3_eqcount_i32; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_lines/$w.json 2> gpurun_out/bench_lines/$w.err
  echo "$w rc=$?"
done
for f in gpurun_out/bench_lines/cfg1*.json gpurun_out/bench_lines/cfg3*.json gpurun_out/bench_lines/cfg0*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['tile'], d['config']['tuning'], round(d['roofline']['frac'],3))
"; done
