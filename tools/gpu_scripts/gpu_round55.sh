#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python tools/hbm_kernels.py 2>&1 | grep -i "gram\|Q R"
timeout 1200 python bench.py --no-cpu > gpurun_out/b55_c3.json 2> gpurun_out/b55_c3.err; echo "bench rc=$?"
grep "^{" gpurun_out/b55_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']))"
