#!/bin/bash
# round 2: column-chunked filter (allreduce of one half overlapped with the other half's tile
# product, BSE200_CHUNK_MIN) with the final real-split kernels, C3 at N = 4 / 2
mkdir -p gpurun_out/r02k
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29601"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29603"
show() { grep "^{" $1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'])"; }
BSE200_CHUNK_MIN=512 timeout 1200 $TR4 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > gpurun_out/r02k/bench_c3_n4_chunk.json 2> gpurun_out/r02k/n4.err; echo "n4 chunk rc=$?"; show gpurun_out/r02k/bench_c3_n4_chunk.json
BSE200_CHUNK_MIN=512 timeout 1200 $TR2 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e > gpurun_out/r02k/bench_c3_n2_chunk.json 2> gpurun_out/r02k/n2.err; echo "n2 chunk rc=$?"; show gpurun_out/r02k/bench_c3_n2_chunk.json
