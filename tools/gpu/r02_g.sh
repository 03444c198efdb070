#!/bin/bash
# round 2, call g (4 GPUs): NCCL dist parity at N=4 (one-tile plane storage), C3 at N=4, C4 at N=4,
# and the 8-GPU 2 x 4 grid as 8 ranks on 4 GPUs (gloo) at C3 size: functional + memory headroom
mkdir -p gpurun_out/r02g
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521"
timeout 900 $TR4 tools/dist_check.py > gpurun_out/r02g/dist_check_n4.txt 2>&1; echo "dist_check4 rc=$?"
grep -E "OK|FAIL" gpurun_out/r02g/dist_check_n4.txt | head -12
timeout 1800 $TR4 bench.py --gpus 4 --steps 2 --warmup 1 > gpurun_out/r02g/bench_c3_n4.json 2> gpurun_out/r02g/bench_c3_n4.err; echo "bench c3 n4 rc=$?"
grep "^{" gpurun_out/r02g/bench_c3_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['memory'], d['solve']['ledger_seconds'])"
timeout 2400 $TR4 bench.py --gpus 4 --config c4 --steps 1 --warmup 0 --no-e2e > gpurun_out/r02g/bench_c4_n4.json 2> gpurun_out/r02g/bench_c4_n4.err; echo "bench c4 n4 rc=$?"
grep "^{" gpurun_out/r02g/bench_c4_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['memory'], d['solve']['iterations'], d['solve']['ledger_seconds'])"
TR8="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29523"
BSE200_DIST_BACKEND=gloo timeout 2400 $TR8 bench.py --gpus 8 --steps 1 --warmup 0 --no-e2e > gpurun_out/r02g/bench_c3_2x4grid_gloo_8ranks_on_4gpus.json 2> gpurun_out/r02g/bench_c3_8ranks.err; echo "8 ranks rc=$?"
grep "^{" gpurun_out/r02g/bench_c3_2x4grid_gloo_8ranks_on_4gpus.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['memory'], d['config']['parallelism'], d['solve']['iterations'], d['solve']['lambda_1'], d['solve']['locked_per_iter'])"
