#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
NG=4
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29518"
timeout 600 $TR tools/dist_check.py > gpurun_out/dist_check_$NG.log 2>&1; echo "dist_check rc=$?"; grep -c OK gpurun_out/dist_check_$NG.log
timeout 900 $TR bench.py --gpus $NG > gpurun_out/b28_c3_n$NG.json 2> gpurun_out/b28_c3_n$NG.err; echo "c3 n$NG rc=$?"
grep "^{" gpurun_out/b28_c3_n$NG.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'])"
timeout 900 python bench.py > gpurun_out/b28_c3_n1.json 2> gpurun_out/b28_c3_n1.err; echo "c3 n1 rc=$?"
grep "^{" gpurun_out/b28_c3_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'], d['roofline']['frac'])"
