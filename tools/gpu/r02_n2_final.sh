#!/bin/bash
# round 2: C3 at N = 2 with the final build
mkdir -p gpurun_out/r02n2
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631"
timeout 1200 $TR2 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02n2/bench_c3_n2.json 2> gpurun_out/r02n2/bench_c3_n2.err; echo "bench n2 rc=$?"
grep "^{" gpurun_out/r02n2/bench_c3_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['clocks'])"
