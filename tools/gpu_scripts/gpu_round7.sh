#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512"
timeout 900 python bench.py --config c3 --steps 1 --warmup 1 --no-cpu > gpurun_out/bench_c3_n1_ev.json 2> gpurun_out/bench_c3_n1_ev.err; echo "c3 n1 rc=$?"
timeout 900 $TR bench.py --gpus $NG --config c3 --steps 1 --warmup 1 > gpurun_out/bench_c3_n${NG}_ev.json 2> gpurun_out/bench_c3_n${NG}_ev.err; echo "c3 n$NG rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/bench_c3_n1_ev.json", "gpurun_out/bench_c3_n2_ev.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, d["value"], d["solve"]["ledger_seconds"])
    ev = d["solve"]["phase_events_s"]
    print(" ", [(p, t) for p, t in ev if p != "filter"])
PY
cat > /tmp/hop3.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.variants(20000, [1200], [3])
PY
python /tmp/hop3.py > gpurun_out/hop3_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:hop_kernel -s 1 -c 1 -o gpurun_out/prof_hop3m_c3 python /tmp/hop3.py > gpurun_out/ncu_hop3.log 2>&1; echo "ncu rc=$?"
