#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x -k "3m or apply_h or filter" > gpurun_out/pytest_3m.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_3m.log
cat > /tmp/t4.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.whole_filter(20000, [1200, 300], [4, 6, 7])
tune_hop.whole_filter(10000, [600, 113], [4, 6, 7])
PY
python /tmp/t4.py > gpurun_out/tune_xsum.log 2>&1; cat gpurun_out/tune_xsum.log
