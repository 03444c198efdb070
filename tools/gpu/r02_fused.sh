#!/bin/bash
# round 2: fused tile product + group reduction over NVLink peer memory (BSE200_FUSED_REDUCE=1)
mkdir -p gpurun_out/r02u
N=${1:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29611"
BSE200_FUSED_REDUCE=1 timeout 600 $TR tools/dist_check.py > gpurun_out/r02u/dist_check_fused_n$N.txt 2>&1; echo "dist_check fused rc=$?"; grep -cE " OK" gpurun_out/r02u/dist_check_fused_n$N.txt; grep -E "FAIL|Error|error" gpurun_out/r02u/dist_check_fused_n$N.txt | head -5
BSE200_FUSED_REDUCE=1 timeout 900 $TR bench.py --gpus $N --steps ${2:-3} --warmup 3 --no-e2e > gpurun_out/r02u/bench_c3_n${N}_fused.json 2> gpurun_out/r02u/bench_n${N}_fused.err; echo "bench fused rc=$?"
grep "^{" gpurun_out/r02u/bench_c3_n${N}_fused.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['solve']['ledger_seconds'], d['parity_vs_reference']['pass'], d['parity_vs_reference']['max_dlambda_rel'])"
tail -3 gpurun_out/r02u/bench_n${N}_fused.err
