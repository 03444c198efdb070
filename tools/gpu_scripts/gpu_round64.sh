#!/bin/bash
# C4 (n = 100k, nev 3000, nex 500) on 4 GPUs with the real-split filter: one timed solve
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29564"
timeout 1500 $TR bench.py --gpus 4 --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r64_c4_n4.json 2> gpurun_out/r64_c4_n4.err; echo "c4 n4 rc=$?"
grep "^{" gpurun_out/r64_c4_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['filter_algorithm'], s['ledger_seconds'], s['iterations'], s['converged'], d['filter_tflops_per_gpu'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']), s['generator_s'])"
grep -i "planes\|warn\|error" gpurun_out/r64_c4_n4.err | head -5
