#!/bin/bash
# split-K real-split kernel: timing per factor at C3 tile shapes, correctness vs the unsplit tile
set -x
cd "$GRAFT_REPO_ROOT"
O=gpurun_out/r02s
mkdir -p $O
for m in 20000 10000; do
  for s in 1 2 3 4 0; do
    BSE200_RS_KSPLIT=$s timeout 300 python tools/rs_bench.py $m 1200,900,600,300,200,100 97,90 > $O/rs_m${m}_s${s}.jsonl 2> $O/rs_m${m}_s${s}.err
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -m gpu > $O/pytest.log 2>&1
