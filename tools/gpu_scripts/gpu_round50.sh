#!/bin/bash
mkdir -p gpurun_out
T0=$SECONDS; timeout 1800 python bench.py > gpurun_out/b50_default.json 2> gpurun_out/b50_default.err; echo "bench rc=$? wall $((SECONDS - T0)) s"
grep "^{" gpurun_out/b50_default.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['cpu_baseline'], d['roofline']['frac'], d['clocks'])"
T0=$SECONDS; timeout 1800 python bench.py --impl reference > gpurun_out/b50_ref.json 2> gpurun_out/b50_ref.err; echo "ref rc=$? wall $((SECONDS - T0)) s"; tail -1 gpurun_out/b50_ref.json | cut -c1-300
