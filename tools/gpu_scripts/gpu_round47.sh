#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -q -m gpu -k "c64 or mixed" 2>&1 | tail -3
cat > /tmp/c64speed.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.c64_filter(20000, [1200, 300])
tune_hop.c64_filter(10000, [600, 113])
PY
for P in 1 0; do echo "BSE200_C64_PAIR=$P"; BSE200_C64_PAIR=$P timeout 300 python /tmp/c64speed.py 2>&1 | tail -4; done
