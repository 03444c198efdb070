#!/bin/bash
# round 2, call h (4 GPUs): final build (split-K + ragged last column tile) at N = 4 / 2 (C3)
mkdir -p gpurun_out/r02h
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29593"
show() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'], d['clocks'])"; }
timeout 1500 $TR4 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02h/bench_c3_n4.json 2> gpurun_out/r02h/bench_c3_n4.err; echo "bench n4 rc=$?"; show gpurun_out/r02h/bench_c3_n4.json
timeout 1500 $TR2 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r02h/bench_c3_n2.json 2> gpurun_out/r02h/bench_c3_n2.err; echo "bench n2 rc=$?"; show gpurun_out/r02h/bench_c3_n2.json
