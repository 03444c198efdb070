#!/bin/bash
# final check after "sum planes only where the real-split planes are unavailable": GPU suite, smoke,
# dist_check at N = 2, default bench line (N = 1)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r67_pytest_gpu.log; tail -3 gpurun_out/r67_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r67_smoke.log 2>&1; tail -1 gpurun_out/r67_smoke.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572"
timeout 600 $TR tools/dist_check.py > gpurun_out/r67_dist_check_n2.log 2>&1; echo "dist_check n2 rc=$?"; grep "world" gpurun_out/r67_dist_check_n2.log | tail -10
timeout 900 python bench.py > gpurun_out/r67_bench.json 2> gpurun_out/r67_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r67_bench.json')); print(d['value'], d['e2e']['value'], d['roofline']['achieved'], d['filter_executed_frac_of_fp64_peak'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['clocks'], d['cpu_baseline']['value'])"
