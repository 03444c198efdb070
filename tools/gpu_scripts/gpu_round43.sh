#!/bin/bash
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29538"
BSE200_DIST_BACKEND=gloo timeout 900 $TR tools/dist_check.py > gpurun_out/dist_check_gloo8.log 2>&1; echo "dist_check gloo 8 ranks on 4 GPUs rc=$?"
grep "world" gpurun_out/dist_check_gloo8.log | tail -8; grep -iE "error|Traceback" gpurun_out/dist_check_gloo8.log | head -5
