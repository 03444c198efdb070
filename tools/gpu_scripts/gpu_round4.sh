#!/bin/bash
mkdir -p gpurun_out
python tools/profile_solve.py c2 > gpurun_out/profile_c2.txt 2>&1; echo "profile rc=$?"
head -60 gpurun_out/profile_c2.txt
# ncu: launch list of the filter microbench, then one full capture of the hop kernel at the C3 shape
cat > /tmp/hop_one.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from bench_hop import run
run(20000, 1200, reps=1)
PY
python /tmp/hop_one.py > gpurun_out/hop_one_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_hop.csv python /tmp/hop_one.py > gpurun_out/ncu_launches.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:hop_kernel -s 2 -c 1 -o gpurun_out/prof_hop_c3 python /tmp/hop_one.py > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
tail -3 gpurun_out/ncu_full.log
