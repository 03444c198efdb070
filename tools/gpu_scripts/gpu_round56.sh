#!/bin/bash
mkdir -p gpurun_out
timeout 2700 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/b56_c4_n1.json 2> gpurun_out/b56_c4_n1.err; echo "c4 n1 rc=$?"
grep "^{" gpurun_out/b56_c4_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], s['ledger_seconds'], s['iterations'], s['converged'], d['filter_tflops_per_gpu'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']))"
grep -i "sum planes\|warn\|error" gpurun_out/b56_c4_n1.err | head -5
nvidia-smi --query-gpu=memory.total --format=csv
