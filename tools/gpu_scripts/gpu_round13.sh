#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x -k "3m or apply_h or filter" > gpurun_out/pytest_3m.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_3m.log
cat > /tmp/t3.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.variants(20000, [1200, 300], [4, 3, 6, 61, 62, 63])
tune_hop.variants(10000, [600, 113], [4, 6, 61, 62, 63])
PY
python /tmp/t3.py > gpurun_out/tune_3ms.log 2>&1; cat gpurun_out/tune_3ms.log
