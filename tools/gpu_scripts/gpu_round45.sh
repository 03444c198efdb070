#!/bin/bash
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e"
$CMD > gpurun_out/b45_plain.json 2> gpurun_out/b45_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_bench_c3.csv $CMD > gpurun_out/b45_ncu.log 2>&1; echo "ncu rc=$?"
python - <<'PY' | tee gpurun_out/ncu_launch_shares.txt
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/ncu_launches_bench_c3.csv")) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = collections.Counter(); cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0][:90]
    v = float(r[14].replace(",", ""))
    unit = r[13]
    v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
    tot[name] += v; cnt[name] += 1
allt = sum(tot.values())
print(f"launches {len(rows)}, total kernel time {allt:.1f} ms")
for name, t in tot.most_common(15):
    print(f"{t:12.1f} ms {100 * t / allt:6.2f}%  x{cnt[name]:4d}  {name}")
PY
gzip -f gpurun_out/ncu_launches_bench_c3.csv
