#!/bin/bash
# round 2: the plan with the < 20-waves rule at m = 10k / 20k, then C3 at N = 4 (and N = 1 below)
mkdir -p gpurun_out/r02v2
timeout 300 python tools/rs_bench.py 10000 1200,1133,810,642,502,266,220 90 > gpurun_out/r02v2/rs_m10k.jsonl 2>&1
timeout 300 python tools/rs_bench.py 20000 1200,1133,810,642,502,266,220 90 > gpurun_out/r02v2/rs_m20k.jsonl 2>&1
python - <<'PY'
import json
for f in ("rs_m10k", "rs_m20k"):
    print(f, " ".join(f"{r['k']}:{(r['fwd_frac'] + r['trans_frac']) / 2:.4f}" for r in map(json.loads, (l for l in open(f"gpurun_out/r02v2/{f}.jsonl") if l.startswith("{")))))
PY
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621"
timeout 1500 $TR4 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02v2/bench_c3_n4.json 2> gpurun_out/r02v2/bench_c3_n4.err; echo "bench n4 rc=$?"
grep "^{" gpurun_out/r02v2/bench_c3_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['clocks'])"
