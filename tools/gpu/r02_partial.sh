#!/bin/bash
# round 2: skip the 8-column fragments beyond k in the last column tile (ragged widths): per-k
# timing at the solve's widths, tile bitwise tests, split-K tests
mkdir -p gpurun_out/r02p
timeout 600 python tools/rs_bench.py 20000 1200,1133,810,642,502,266,220,100 97,90 > gpurun_out/r02p/rs_m20k.jsonl 2>&1; echo "rs20k rc=$?"
timeout 600 python tools/rs_bench.py 10000 1200,1133,810,642,502,266,220 90 > gpurun_out/r02p/rs_m10k.jsonl 2>&1; echo "rs10k rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/r02p/rs_m20k.jsonl", "gpurun_out/r02p/rs_m10k.jsonl"):
    for l in open(f):
        if l.startswith("{"):
            r = json.loads(l); print(f[-12:], r["m"], r["k"], r["code"], round(r["fwd_ms"], 3), round(r["fwd_frac"], 4), round(r["trans_frac"], 4), r["bitwise_as_first_code"])
PY
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -k "rs or split or transposed or tile" > gpurun_out/r02p/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02p/pytest.log
