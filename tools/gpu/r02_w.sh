#!/bin/bash
# round 2, call w (4 GPUs): final multi-GPU numbers with the BK = 32 tile: C3 at N = 4 / 2 (20 steps,
# as the driver runs them), NCCL parity at N = 4, the 2 x 4 grid functional run (8 ranks, gloo)
mkdir -p gpurun_out/r02w
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29573"
TR8="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29575"
timeout 900 $TR4 tools/dist_check.py > gpurun_out/r02w/dist_check_n4.txt 2>&1; echo "dist_check4 rc=$?"; grep -cE " OK" gpurun_out/r02w/dist_check_n4.txt; grep FAIL gpurun_out/r02w/dist_check_n4.txt
for N in 4 2; do
  TR=$([ $N = 4 ] && echo "$TR4" || echo "$TR2")
  timeout 2400 $TR bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r02w/bench_c3_n$N.json 2> gpurun_out/r02w/bench_c3_n$N.err; echo "bench n$N rc=$?"
  grep "^{" gpurun_out/r02w/bench_c3_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['clocks'])"
done
BSE200_DIST_BACKEND=gloo timeout 2400 $TR8 bench.py --gpus 8 --steps 1 --warmup 0 --no-e2e > gpurun_out/r02w/bench_c3_2x4grid_gloo_8ranks_on_4gpus.json 2> gpurun_out/r02w/bench_c3_8ranks.err; echo "8 ranks rc=$?"
grep "^{" gpurun_out/r02w/bench_c3_2x4grid_gloo_8ranks_on_4gpus.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['memory'], d['config']['parallelism'], d['solve']['iterations'], d['parity_vs_reference']['pass'])"
