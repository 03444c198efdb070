#!/bin/bash
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29581"
BSE200_DIST_BACKEND=gloo timeout 1500 $TR bench.py --gpus 8 --config c2 --steps 1 --warmup 3 > gpurun_out/b53_c2_gloo8.json 2> gpurun_out/b53_c2_gloo8.err; echo "bench c2 8 ranks/4 GPUs gloo rc=$?"
grep "^{" gpurun_out/b53_c2_gloo8.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['n_gpus'], d['value'], d['e2e']['value'], s['iterations'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']), d['config']['parallelism'])"
grep -iE "error|Traceback" gpurun_out/b53_c2_gloo8.err | head -5
