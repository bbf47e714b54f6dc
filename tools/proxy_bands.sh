#!/bin/bash
# Rank 0's row band of an N-way split, timed alone on one GPU (bench.py
# --proxy-band N): the per-rank work of an N-GPU run, device-resident and
# end to end, for configs 4 and 3. Not a multi-GPU measurement.
out=gpurun_out/r02/proxy
mkdir -p $out
for n in 2 4 8; do
  python bench.py --workload cfg4_discount_f64 --steps 5 --warmup 3 --no-cpu --proxy-band $n > $out/cfg4_band_of_$n.json 2> $out/cfg4_band_of_$n.err
  echo "cfg4 band of $n rc=$?"
done
for w in cfg3_sqdiff_f32 cfg3_eqcount_i32; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --proxy-band 8 > $out/${w}_band_of_8.json 2> $out/${w}_band_of_8.err
  echo "$w band of 8 rc=$?"
done
