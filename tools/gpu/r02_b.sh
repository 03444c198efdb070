#!/bin/bash
# round 2, call b (2 GPUs): GPU tests, NCCL dist parity at N=2, C3 bench at N=2 (one-tile storage)
mkdir -p gpurun_out/r02b
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02b/pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02b/pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 900 $TR tools/dist_check.py > gpurun_out/r02b/dist_check_n2.txt 2>&1; echo "dist_check rc=$?"
grep -E "OK|FAIL|world" gpurun_out/r02b/dist_check_n2.txt | head -20
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT timeout 1500 $TR bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/r02b/bench_c3_n2.json 2> gpurun_out/r02b/bench_c3_n2.err; echo "bench n2 rc=$?"
grep "^{" gpurun_out/r02b/bench_c3_n2.json | tail -c 2500; grep -c "NCCL INFO" gpurun_out/r02b/bench_c3_n2.json; tail -3 gpurun_out/r02b/bench_c3_n2.err
