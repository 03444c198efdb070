#!/bin/bash
# C3 with the opt-in mixed-precision policy (first filters complex64 on tcgen05, then the real-split FP64 filter)
mkdir -p gpurun_out
timeout 900 python bench.py --config c3mixed --no-cpu > gpurun_out/r66_c3mixed.json 2> gpurun_out/r66_c3mixed.err; echo "c3mixed rc=$?"
grep "^{" gpurun_out/r66_c3mixed.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['solve']; print(d['value'], d['e2e']['value'], s['ledger_seconds'], s['iterations'], s['locked_per_iter'], s['filter_precision_per_iter'], repr(s['lambda_1']), repr(s['lambda_nev']), s['max_residual'])"
