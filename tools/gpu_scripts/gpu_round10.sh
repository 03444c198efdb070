#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29515"
BSE200_TIMING=1 timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > gpurun_out/b10_c3_n1.json 2> gpurun_out/b10_c3_n1.err; echo "c3 n1 rc=$?"
grep bse200 gpurun_out/b10_c3_n1.err | tail -120 > gpurun_out/b10_timing_n1.txt
BSE200_TIMING=1 timeout 900 $TR bench.py --gpus $NG --config c3 --steps 1 --warmup 1 > gpurun_out/b10_c3_n$NG.json 2> gpurun_out/b10_c3_n$NG.err; echo "c3 n$NG rc=$?"
grep -E "^\[dist|^\[bse200" gpurun_out/b10_c3_n$NG.json | tail -300 > gpurun_out/b10_timing_n$NG.txt
python - <<'PY'
import json
for f in ["gpurun_out/b10_c3_n1.json", "gpurun_out/b10_c3_n2.json"]:
    try:
        d = json.loads([l for l in open(f).read().strip().splitlines() if l.startswith("{")][-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["e2e"]["value"], d["solve"]["ledger_seconds"])
PY
