# ncu (pipe utilisation, issue, DRAM) of each remaining config's winning kernel
mkdir -p gpurun_out/ncu_cfg
M=sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active
run() {  # tag workload tile regex [extra]
  timeout 900 ncu --metrics $M --clock-control none -k "regex:$4" -c 1 --csv --log-file gpurun_out/ncu_cfg/$1.csv \
    python bench.py --workload $2 --steps 1 --warmup 1 --no-cpu --no-e2e --tile $3 $5 > gpurun_out/ncu_cfg/$1.log 2>&1
  echo "$1 rc=$?"
}
run cfg1_boost_f32 cfg1_boost_f32 boost_f32_32x128_t4x4_w8x1 mmlt_tile_kernel
run cfg1_boost_f64 cfg1_boost_f64 boost_f64_16x128_t4x4_w4x1 mmlt_tile_kernel
run cfg3_sqdiff_f32 cfg3_sqdiff_f32 sqdiff_f32_32x128_t4x4_w8x1 mmlt_tile_kernel
run cfg2_gemm_f64 cfg2_gemm_f64 gemm_f64_64x128_dmma_w32x32_c2x4 dmma_gemm_kernel
run cfg0_discount_f64 cfg0_discount_f64 discount_f64_16x128_t4x4_w4x1 mmlt_tile_kernel
