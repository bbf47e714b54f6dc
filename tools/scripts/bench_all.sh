# every BASELINE config through bench.py (device-resident value, e2e, roofline,
# reference CPU baseline), one JSON line each under gpurun_out/bench_lines/
mkdir -p gpurun_out/bench_lines
for w in cfg0_discount_f64 cfg1_boost_f32 cfg1_boost_f64 cfg2_gemm_f64 cfg2_gemm_f32 cfg3_sqdiff_f32; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_lines/$w.json 2> gpurun_out/bench_lines/$w.err
  echo "$w rc=$?"
done
timeout 900 python bench.py --workload cfg2_gemm_f64 --f64-emulation --steps 10 --warmup 3 > gpurun_out/bench_lines/cfg2_gemm_f64_f64emulation.json 2> gpurun_out/bench_lines/cfg2_gemm_f64_f64emulation.err
echo "cfg2 emulation rc=$?"
for f in gpurun_out/bench_lines/*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print('$f'.split('/')[-1], round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['tile'], round(d['roofline']['frac'],3), d['clocks'])
"; done
