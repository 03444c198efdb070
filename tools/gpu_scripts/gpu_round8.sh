#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29513"
timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > gpurun_out/b8_c3_n1.json 2> gpurun_out/b8_c3_n1.err; echo "c3 n1 rc=$?"
timeout 900 $TR bench.py --gpus $NG --config c3 --steps 1 --warmup 1 > gpurun_out/b8_c3_n$NG.json 2> gpurun_out/b8_c3_n$NG.err; echo "c3 n$NG rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/b8_c3_n1.json", "gpurun_out/b8_c3_n2.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["e2e"]["value"], d["solve"]["ledger_seconds"], d["clocks"])
    ev = d["solve"]["phase_events_s"]
    print(" ", [(p, t) for p, t in ev if p != "filter"])
PY
