
python bench.py --workload cfg0_discount_f64 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/c0_tuned.json 2>gpurun_out/c0_tuned.err
for t in "discount_f64_48x128_theta_t6x4_w8x1 208" "discount_f64_32x128_t4x4_w8x1 208" "discount_f64_48x128_theta_t6x4_w8x1 256" "discount_f64_48x128_theta_t6x4_w8x1 512" "discount_f64_48x128_theta_t6x4_w8x1 0" "discount_f64_64x128_theta_t8x4_w8x1 256" "discount_f64_32x128_t4x4_w8x1 256"; do
  set -- $t
  python bench.py --workload cfg0_discount_f64 --steps 20 --warmup 3 --no-cpu --no-e2e --tile $1 --kc $2 > gpurun_out/c0_$1_$2.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c0_$1_$2.json')); print('$1 $2', round(d['value']), d['step_ms_rank0'])"
done
python -c "import json; d=json.load(open('gpurun_out/c0_tuned.json')); print('tuned', round(d['value']), d['config']['tile'], d['config']['split_k_kc'], d['step_ms_rank0'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg0_theta.csv python bench.py --workload cfg0_discount_f64 --steps 3 --warmup 3 --no-cpu --no-e2e --no-verify --tile discount_f64_48x128_theta_t6x4_w8x1 --kc 256 > /dev/null 2>&1
echo ncu rc=$?
