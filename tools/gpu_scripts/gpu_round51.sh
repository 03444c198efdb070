#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "bitwise or 3m" 2>&1 | tail -3
cat > /tmp/tune.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.whole_filter(20000, [1200, 300], [86, 89, 82, 90])
tune_hop.whole_filter(10000, [600, 113], [86, 89, 82, 90])
PY
timeout 600 python /tmp/tune.py 2>&1 | tail -16
