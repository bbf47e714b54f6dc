# full GPU test suite, the default bench line, the reference arm, and the
# launch list of the bench command (winner pinned), for profiles/
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_cfg4.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --tile discount_f64_96x128_theta_t8x4_w12x1 > gpurun_out/ncu_bench.log 2>&1; echo ncu rc=$?
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/launches_cfg4.csv")) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
tot = collections.Counter(); n = collections.Counter()
for r in rows[1:]:
    try: v = float(r[vi].replace(",", ""))
    except ValueError: continue
    tot[r[ki][:90]] += v; n[r[ki][:90]] += 1
s = sum(tot.values())
for k, v in tot.most_common(8): print(f"{100*v/s:6.2f}%  {n[k]:4d}x  {v/n[k]/1e6:10.3f} ms  {k}")
PY
