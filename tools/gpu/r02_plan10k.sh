#!/bin/bash
# round 2: split-K factor vs the plan at the 2 x 2 grid's tile (m = 10k) and the C3 solve's widths
mkdir -p gpurun_out/r02q
for s in 0 1 2 3 4; do
  BSE200_RS_KSPLIT=$s timeout 300 python tools/rs_bench.py 10000 1200,1133,810,642,502,266,220 90 > gpurun_out/r02q/rs_m10k_s$s.jsonl 2>&1
done
python - <<'PY'
import json
rows = {}
for s in (0, 1, 2, 3, 4):
    for l in open(f"gpurun_out/r02q/rs_m10k_s{s}.jsonl"):
        if l.startswith("{"):
            r = json.loads(l); rows.setdefault(r["k"], {})[s] = (r["fwd_frac"] + r["trans_frac"]) / 2
for k, d in rows.items():
    print(k, " ".join(f"s{s}={d[s]:.4f}" for s in sorted(d)))
PY
