#!/bin/bash
# real-split filter on the 2D grid: GPU suite (1 GPU), dist_check at N = 2 (NCCL) and the
# 2 x 4 grid as 8 gloo ranks, then the C3 bench at N = 2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r62_pytest_gpu.log; tail -3 gpurun_out/r62_pytest_gpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542"
timeout 600 $TR tools/dist_check.py > gpurun_out/r62_dist_check_n2.log 2>&1; echo "dist_check n2 rc=$?"; grep "world" gpurun_out/r62_dist_check_n2.log | tail -10
TR8="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29548"
BSE200_DIST_BACKEND=gloo timeout 900 $TR8 tools/dist_check.py > gpurun_out/r62_dist_check_8gloo.log 2>&1; echo "dist_check 8 gloo ranks rc=$?"; grep "world" gpurun_out/r62_dist_check_8gloo.log | tail -10
timeout 1500 $TR bench.py --gpus 2 > gpurun_out/r62_bench_c3_n2.json 2> gpurun_out/r62_bench_c3_n2.err; echo "bench n2 rc=$?"
grep "^{" gpurun_out/r62_bench_c3_n2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], d['filter_algorithm'], d['roofline']['achieved'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'])"
tail -3 gpurun_out/r62_bench_c3_n2.err
timeout 900 python bench.py --steps 1 --warmup 3 > gpurun_out/r62_bench_c3_n1.json 2> gpurun_out/r62_bench_c3_n1.err
python -c "import json; d=json.load(open('gpurun_out/r62_bench_c3_n1.json')); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['locked_per_iter'])"
