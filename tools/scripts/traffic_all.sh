# DRAM bytes per launch of each config's winning kernel (ncu launch list with
# the winner pinned), for the roofline.traffic field
mkdir -p gpurun_out/traffic
run() {  # tag workload tile kernel-regex [extra]
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k "regex:$4" -c 6 --csv --log-file gpurun_out/traffic/$1.csv \
    python bench.py --workload $2 --steps 1 --warmup 1 --no-cpu --no-e2e --tile $3 $5 > gpurun_out/traffic/$1.log 2>&1
  echo "$1 rc=$?"
}
run cfg0_discount_f64 cfg0_discount_f64 discount_f64_16x128_t4x4_w4x1 mmlt_tile_kernel
run cfg1_boost_f32 cfg1_boost_f32 boost_f32_32x128_t4x4_w8x1 mmlt_tile_kernel
run cfg1_boost_f64 cfg1_boost_f64 boost_f64_16x128_t4x4_w4x1 mmlt_tile_kernel
run cfg2_gemm_f64 cfg2_gemm_f64 gemm_f64_64x128_dmma_w32x32_c2x4 dmma_gemm_kernel
run cfg3_sqdiff_f32 cfg3_sqdiff_f32 sqdiff_f32_32x128_t4x4_w8x1 mmlt_tile_kernel
run cfg2_gemm_f64_f64emulation cfg2_gemm_f64 gemm_f64_128x64_tcgen05_ozaki_i8 ozaki_gemm_kernel --f64-emulation
