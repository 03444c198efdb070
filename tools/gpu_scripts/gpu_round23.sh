#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/t6.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.c64_filter(20000, [1200, 300])
tune_hop.c64_filter(10000, [600, 113])
PY
timeout 600 python /tmp/t6.py > gpurun_out/c64_speed.log 2>&1; echo "rc=$?"; cat gpurun_out/c64_speed.log
timeout 900 python bench.py --config c3c64 --steps 1 --warmup 1 --no-cpu > gpurun_out/b23_c3c64.json 2> gpurun_out/b23_c3c64.err; echo "c3c64 rc=$?"
grep "^{" gpurun_out/b23_c3c64.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['filter_tflops_per_gpu'], d['solve']['locked_per_iter'], d['solve']['lambda_1'], d['solve']['lambda_nev'])"
tail -3 gpurun_out/b23_c3c64.err
