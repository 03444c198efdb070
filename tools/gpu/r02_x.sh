#!/bin/bash
# round 2, call x (4 GPUs): the 8-GPU 2 x 4 grid as 8 ranks on 4 GPUs (gloo collectives, CUDA
# kernels): golden cases + C1 (dist_check) and a C3 solve (functional: memory, trace, parity)
mkdir -p gpurun_out/r02x
TR8="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29581"
BSE200_DIST_BACKEND=gloo timeout 1500 $TR8 tools/dist_check.py > gpurun_out/r02x/dist_check_2x4_gloo_8ranks.txt 2>&1; echo "dist_check8 rc=$?"
grep -E "OK|FAIL" gpurun_out/r02x/dist_check_2x4_gloo_8ranks.txt | head -12
BSE200_DIST_BACKEND=gloo timeout 2400 $TR8 bench.py --gpus 8 --steps 1 --warmup 0 --no-e2e > gpurun_out/r02x/bench_c3_2x4grid_gloo_8ranks_on_4gpus.json 2> gpurun_out/r02x/bench_c3_8ranks.err; echo "8 ranks rc=$?"
grep "^{" gpurun_out/r02x/bench_c3_2x4grid_gloo_8ranks_on_4gpus.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['memory'], d['config']['parallelism'], d['solve']['iterations'], d['parity_vs_reference'])"
