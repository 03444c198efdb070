#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-2}
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511"
timeout 600 $TR tools/dist_check.py > gpurun_out/dist_check_$NG.log 2>&1; echo "dist_check rc=$?"
grep -E "world|Error|error" gpurun_out/dist_check_$NG.log | head -20
timeout 900 $TR bench.py --gpus $NG --config c2 --steps 1 --warmup 1 > gpurun_out/bench_c2_n$NG.json 2> gpurun_out/bench_c2_n$NG.err; echo "c2 n$NG rc=$?"
cat gpurun_out/bench_c2_n$NG.json; tail -3 gpurun_out/bench_c2_n$NG.err
timeout 1200 $TR bench.py --gpus $NG --config c3 --steps 1 --warmup 1 > gpurun_out/bench_c3_n$NG.json 2> gpurun_out/bench_c3_n$NG.err; echo "c3 n$NG rc=$?"
cat gpurun_out/bench_c3_n$NG.json; tail -3 gpurun_out/bench_c3_n$NG.err
