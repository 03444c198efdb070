#!/bin/bash
# launch list of one C3 solve in the final state (bench --steps 1 --warmup 0 --no-cpu) and ncu of the
# narrow real-split tile (k = 300)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 0 --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r68_ncu_launches_bench_c3.csv $CMD > gpurun_out/r68_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python - <<'PY' | tee gpurun_out/r68_ncu_launch_shares.txt
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/r68_ncu_launches_bench_c3.csv")) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = collections.Counter(); cnt = collections.Counter()
for r in rows:
    name = r[4].split("(")[0][:80]
    v = float(r[14].replace(",", ""))
    unit = r[13]
    v = v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(unit, 1.0)
    tot[name] += v; cnt[name] += 1
allt = sum(tot.values())
print(f"launches {len(rows)}, total kernel time {allt:.1f} ms (one timed C3 solve + the e2e solve)")
for name, t in tot.most_common(15):
    print(f"{t:12.1f} ms {100 * t / allt:6.2f}%  x{cnt[name]:4d}  {name}")
PY
gzip -f gpurun_out/r68_ncu_launches_bench_c3.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hop_rs_tma_kernel -c 1 -o gpurun_out/r68_ncu_rs_narrow \
  python tools/tune_rs.py 20000 300 94 > gpurun_out/r68_ncu_narrow.log 2>&1; echo "ncu narrow rc=$?"
