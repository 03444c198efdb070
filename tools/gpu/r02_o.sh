#!/bin/bash
# round 2, call o (1 GPU): the driver's own sequence -- reference arm, our arm (20 steps), GPU tests,
# smoke -- on the final code
mkdir -p gpurun_out/r02o
timeout 3000 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02o/ref1.out 2> gpurun_out/r02o/ref1.err; echo "ref rc=$?"
tail -c 600 gpurun_out/r02o/ref1.out
timeout 3600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02o/n1.out 2> gpurun_out/r02o/n1.err; echo "ours rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02o/n1.out').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline'], d['solve']['ledger_seconds'], d['cpu_baseline']['value'], d['parity_vs_reference']['pass'], d['clocks'])"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02o/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02o/pytest.log
timeout 300 python __graft_entry__.py > gpurun_out/r02o/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02o/smoke.log
