#!/bin/bash
# real-split filter as the default: full GPU suite, smoke, default bench (C3), launch list, ncu of the RS kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r61_pytest_gpu.log
tail -4 gpurun_out/r61_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r61_smoke.log 2>&1; tail -1 gpurun_out/r61_smoke.log
timeout 900 python bench.py > gpurun_out/r61_bench.json 2> gpurun_out/r61_bench.err
python -c "import json; d=json.load(open('gpurun_out/r61_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['filter_executed_frac_of_fp64_peak'], d['solve']['iterations'], d['solve']['locked_per_iter'], d['clocks'])"
# one RS launch at k = 1200 under ncu --set full (tools/tune_rs.py, code 90 only, deg 4)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hop_rs_tma_kernel -c 1 -o gpurun_out/r61_ncu_rs \
  python tools/tune_rs.py 20000 1200 90 > gpurun_out/r61_ncu.log 2>&1
tail -3 gpurun_out/r61_ncu.log
# launch list of one C3 solve (bench with --steps 1 --warmup 0 --no-cpu) and kernel shares
CMD="python bench.py --steps 1 --warmup 0 --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r61_ncu_launches_bench_c3.csv $CMD > gpurun_out/r61_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python - <<'PY' | tee gpurun_out/r61_ncu_launch_shares.txt
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/r61_ncu_launches_bench_c3.csv")) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = collections.Counter(); cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0][:80]
    v = float(r[14].replace(",", ""))
    unit = r[13]
    v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
    tot[name] += v; cnt[name] += 1
allt = sum(tot.values())
print(f"launches {len(rows)}, total kernel time {allt:.1f} ms")
for name, t in tot.most_common(15):
    print(f"{t:12.1f} ms {100 * t / allt:6.2f}%  x{cnt[name]:4d}  {name}")
PY
gzip -f gpurun_out/r61_ncu_launches_bench_c3.csv
