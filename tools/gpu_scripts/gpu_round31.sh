#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/c64_diag.py > gpurun_out/c64_diag.log 2>&1; echo "rc=$?"; grep -v Warn gpurun_out/c64_diag.log
timeout 600 python -m pytest tests -q -m gpu -x -k "c64 or mixed" > gpurun_out/pytest_c64.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c64.log
cat > /tmp/t8.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.c64_filter(20000, [1200, 300])
tune_hop.c64_filter(10000, [600, 113])
PY
timeout 600 python /tmp/t8.py 2>&1 | grep c64
