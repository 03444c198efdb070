#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x -k "3m or filter or pchb" > gpurun_out/pytest_3m.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_3m.log
cat > /tmp/t5.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.whole_filter(20000, [1200, 300], [6, 9, 91, 92])
tune_hop.whole_filter(10000, [600, 113], [6, 9, 91, 92])
PY
python /tmp/t5.py > gpurun_out/tune_ahead.log 2>&1; cat gpurun_out/tune_ahead.log
