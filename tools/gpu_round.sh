#!/bin/bash
# One GPU pass over every BASELINE bench line plus a keyed ncu capture of
# each winner (run under gpurun; one GPU). Outputs in gpurun_out/r02/.
#   bash tools/gpu_round.sh [workload ...]
set -u
out=gpurun_out/r02
mkdir -p $out/bench_lines
wls=${*:-"cfg4_discount_f64 cfg0_discount_f64 cfg1_boost_f32 cfg1_boost_f64 cfg2_gemm_f64 cfg2_gemm_f32 cfg3_sqdiff_f32 cfg3_eqcount_i32"}
for w in $wls; do
  python bench.py --workload $w --steps 10 --warmup 3 > $out/bench_lines/$w.json 2> $out/bench_lines/$w.err
  echo "$w bench rc=$?"
done
python bench.py --workload cfg2_gemm_f64 --steps 10 --warmup 3 --f64-emulation > $out/bench_lines/cfg2_gemm_f64_f64emulation.json 2> $out/bench_lines/cfg2_gemm_f64_f64emulation.err
for w in $wls; do
  read tile kc iters rx < <(python - "$out/bench_lines/$w.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
c = d["config"]; t = c["tile"] or ""
rx = ("mmlt_tile_kernel<amltk::th::BodyTheta" if "_theta_" in t else "BodySwarEq" if "_swar_" in t else
      "tf32x3_gemm_kernel" if "tcgen05" in t else "ozaki_gemm_kernel" if "ozaki" in t else
      "dmma_gemm_kernel" if "dmma" in t else "mmlt_tile_kernel")
print(t, c["split_k_kc"] or 0, c["M"] * c["N"] * c["K"], rx)
PY
)
  [ -z "$tile" ] && continue
  mkdir -p gpurun_out/keyed
  bash tools/capture_keyed.sh r02 $w $tile "$rx" $iters --kc $kc
done
