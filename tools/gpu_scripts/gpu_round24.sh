#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
cat > /tmp/hop3m.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.whole_filter(20000, [1200], [6], deg=2)
PY
cat > /tmp/c64one.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.c64_filter(20000, [1200], deg=2)
PY
python /tmp/hop3m.py > gpurun_out/hop3m_plain.log 2>&1 && python /tmp/c64one.py > gpurun_out/c64one_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hop_kernel -s 1 -c 1 -o gpurun_out/prof_hop3m_code6 python /tmp/hop3m.py > gpurun_out/ncu_hop3m.log 2>&1; echo "ncu hop rc=$?"
ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/prof_c64_step python /tmp/c64one.py > gpurun_out/ncu_c64.log 2>&1; echo "ncu c64 rc=$?"
