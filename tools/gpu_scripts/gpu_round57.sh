#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
T0=$SECONDS; timeout 1800 python bench.py > gpurun_out/b57_default.json 2> gpurun_out/b57_default.err; echo "bench rc=$? wall $((SECONDS - T0)) s"
grep "^{" gpurun_out/b57_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['cpu_baseline']['value'], d['roofline']['frac'], d['filter_executed_frac_of_fp64_peak'], d['gpu_launches'], d['clocks'])"
