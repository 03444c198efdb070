#!/bin/bash
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -q -m gpu -k "tmaw64" 2>&1 | tail -3
cat > /tmp/tune.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
for m, ks in ((20000, [1200, 300]), (10000, [600, 113])):
    tune_hop.whole_filter(m, ks, [82, 86, 87])
PY
timeout 900 python /tmp/tune.py 2>&1 | tee gpurun_out/tune_mb.txt | tail -20
