#!/bin/bash
# configs[4] B = 0 at C3 in the final state (3M kernel with the B half skipped; the real-split planes are not built)
mkdir -p gpurun_out
timeout 900 python bench.py --config c3b0 --no-cpu > gpurun_out/r69_c3b0.json 2> gpurun_out/r69_c3b0.err; echo "c3b0 rc=$?"
grep "^{" gpurun_out/r69_c3b0.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], d['filter_algorithm'], d['roofline']['achieved'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'])"
