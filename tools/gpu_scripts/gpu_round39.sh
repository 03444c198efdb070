#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log; grep -E "FAIL|Error" gpurun_out/pytest_gpu.log | head -10
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --no-cpu > gpurun_out/b39_c3.json 2> gpurun_out/b39_c3.err; echo "bench rc=$?"
grep "^{" gpurun_out/b39_c3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['solve']['ledger_seconds'], d['solve']['iterations'], d['solve']['locked_per_iter'], d['roofline']['achieved'])"
cat > /tmp/hop86.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.whole_filter(20000, [1200], [86], deg=2)
PY
python /tmp/hop86.py > gpurun_out/hop86_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hop3m_tma_kernel -s 1 -c 1 -o gpurun_out/prof_hop3m_tma86 python /tmp/hop86.py > gpurun_out/ncu_hop86.log 2>&1; echo "ncu rc=$?"
