#!/bin/bash
cat > /tmp/t7.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.whole_filter(20000, [1200, 300], [6, 64, 65, 66])
tune_hop.whole_filter(10000, [600, 113], [6, 64, 65, 66])
PY
python /tmp/t7.py 2>&1 | grep filter
