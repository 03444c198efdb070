#!/bin/bash
cat > /tmp/tune.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
for rep in range(1):
    tune_hop.whole_filter(20000, [1200], [86, 91, 92])
PY
timeout 600 python /tmp/tune.py 2>&1 | tail -4
