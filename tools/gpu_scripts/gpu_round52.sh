#!/bin/bash
cat > /tmp/c64one.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.c64_filter(20000, [1200], deg=2)
PY
python /tmp/c64one.py > gpurun_out/c64one_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 1 -c 1 -o gpurun_out/prof_c64_pair python /tmp/c64one.py > gpurun_out/ncu_c64_pair.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/c64one_plain.log
