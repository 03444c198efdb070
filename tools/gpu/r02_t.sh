#!/bin/bash
# round 2, call t (4 GPUs): final multi-GPU numbers with the 4-warp tile: NCCL parity at N=4, C3 at
# N = 4 / 2, C4 at N = 4, C4 on one GPU (planes only)
mkdir -p gpurun_out/r02t
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29563"
timeout 900 $TR4 tools/dist_check.py > gpurun_out/r02t/dist_check_n4.txt 2>&1; echo "dist_check4 rc=$?"; grep -cE " OK" gpurun_out/r02t/dist_check_n4.txt; grep FAIL gpurun_out/r02t/dist_check_n4.txt
for N in 4 2; do
  TR=$([ $N = 4 ] && echo "$TR4" || echo "$TR2")
  timeout 1800 $TR bench.py --gpus $N --steps 3 --warmup 1 > gpurun_out/r02t/bench_c3_n$N.json 2> gpurun_out/r02t/bench_c3_n$N.err; echo "bench n$N rc=$?"
  grep "^{" gpurun_out/r02t/bench_c3_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['nccl'], d['parity_vs_reference']['pass'])"
done
grep -c "Init COMPLETE" gpurun_out/r02t/bench_c3_n4.err
timeout 2400 $TR4 bench.py --gpus 4 --config c4 --steps 1 --warmup 0 --no-e2e > gpurun_out/r02t/bench_c4_n4.json 2> gpurun_out/r02t/bench_c4_n4.err; echo "c4 n4 rc=$?"
grep "^{" gpurun_out/r02t/bench_c4_n4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['memory'], d['solve']['iterations'], d['solve']['lambda_1'])"
timeout 2400 python bench.py --config c4 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/r02t/bench_c4_n1.json 2> gpurun_out/r02t/bench_c4_n1.err; echo "c4 n1 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02t/bench_c4_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['solve']['iterations'], d['solve']['lambda_1'], d['memory'])"
