#!/bin/bash
# ncu metrics of a bench winner, keyed by (workload, tile) for bench.py's
# roofline (run under gpurun, one GPU). The plain command runs first and must
# exit 0; ncu then profiles ONE launch of the kernel matching <regex>. The CSVs
# come back in gpurun_out/keyed/; merge them here with tools/ncu_keyed.py.
#   bash tools/capture_keyed.sh <round> <workload> <tile> <kernel-regex> <iters/launch> [bench args]
set -u
rnd=$1; wl=$2; tile=$3; rx=$4; iters=$5; shift 5
mkdir -p gpurun_out/keyed
tag=${wl}__${tile}
cmd="python bench.py --workload $wl --tile $tile --steps 1 --warmup 1 --no-e2e --no-cpu --no-verify $*"
$cmd > gpurun_out/keyed/$tag.plain.log 2>&1 || { echo "$tag: plain run failed"; exit 1; }
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread"
M="$M,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"
M="$M,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active"
M="$M,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"
M="$M,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active"
M="$M,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum"
timeout 1200 ncu --metrics "$M" --clock-control none --kernel-name-base demangled -k "regex:$rx" -c 1 \
  --csv --page raw --log-file gpurun_out/keyed/$tag.csv $cmd > gpurun_out/keyed/$tag.ncu.log 2>&1
echo "$tag: ncu rc=$?"
