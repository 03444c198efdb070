#!/bin/bash
# round 2, call m (4 GPUs): C3 at N = 4 / 2 with per-rank draw threads; configs[4] variants on 1 GPU
mkdir -p gpurun_out/r02m
TR4="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29553"
for N in 4 2; do
  TR=$([ $N = 4 ] && echo "$TR4" || echo "$TR2")
  timeout 1800 $TR bench.py --gpus $N --steps 3 --warmup 1 > gpurun_out/r02m/bench_c3_n$N.json 2> gpurun_out/r02m/bench_c3_n$N.err; echo "bench n$N rc=$?"
  grep "^{" gpurun_out/r02m/bench_c3_n$N.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'])"
done
for C in c3b0 c3c64 c3mixed; do
  timeout 1200 python bench.py --config $C --steps 2 --warmup 1 --no-cpu > gpurun_out/r02m/bench_${C}_n1.json 2> gpurun_out/r02m/bench_${C}_n1.err; echo "$C rc=$?"
  python -c "import json; d=json.loads(open('gpurun_out/r02m/bench_${C}_n1.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['filter_algorithm'], d['roofline']['frac'], d['solve']['iterations'], d['solve']['lambda_1'], d['solve']['locked_per_iter'])"
done
