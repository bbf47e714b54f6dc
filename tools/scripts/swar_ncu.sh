mkdir -p gpurun_out
W=eqcount_i32_32x256_swar_t4x8_w8x1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:BodySwarEq -s 0 -c 1 -o gpurun_out/swar_cfg3b python bench.py --workload cfg3_eqcount_i32 --steps 1 --warmup 1 --no-cpu --no-e2e --tile $W > gpurun_out/ncu_full_cfg3b.log 2>&1; echo ncu full rc=$?
ncu -i gpurun_out/swar_cfg3b.ncu-rep --page details --csv > gpurun_out/swar_cfg3b_details.csv 2>&1; echo rc=$?
