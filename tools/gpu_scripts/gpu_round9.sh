#!/bin/bash
mkdir -p gpurun_out
NG=${NG:-2}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29514"
BSE200_TIMING=1 timeout 900 python bench.py --config c3 --steps 1 --warmup 0 --no-cpu > gpurun_out/b9_c3_n1.json 2> gpurun_out/b9_c3_n1.err; echo "c3 n1 rc=$?"
grep bse200 gpurun_out/b9_c3_n1.err | head -150 > gpurun_out/b9_timing_n1.txt
BSE200_TIMING=1 timeout 900 $TR bench.py --gpus $NG --config c3 --steps 1 --warmup 0 > gpurun_out/b9_c3_n$NG.json 2> gpurun_out/b9_c3_n$NG.err; echo "c3 n$NG rc=$?"
grep -E "^\[dist|^\[bse200" gpurun_out/b9_c3_n$NG.json | head -300 > gpurun_out/b9_timing_n$NG.txt
python tools/tune_hop.py > /dev/null 2>&1 || true
cat > /tmp/exp.py <<'PY'
import sys; sys.path.insert(0, "tools"); sys.path.insert(0, ".")
import tune_hop
tune_hop.variants(20000, [1200], [4, 3, 35, 32, 36])
PY
python /tmp/exp.py > gpurun_out/exp35.log 2>&1; cat gpurun_out/exp35.log
