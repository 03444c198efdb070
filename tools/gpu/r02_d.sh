#!/bin/bash
# round 2, call d (1 GPU): all GPU tests (triangle Grams, folded defect, incremental basis,
# pipelined RS kernel), RS kernel timing, CPU model check at C2, reference arm + bench at C3
mkdir -p gpurun_out/r02d
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02d/pytest.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|Error" gpurun_out/r02d/pytest.log | tail -12
timeout 600 python tools/rs_bench.py 20000 1200,300,100 > gpurun_out/r02d/rs_bench.txt 2>&1; echo "rs_bench rc=$?"; cat gpurun_out/r02d/rs_bench.txt
timeout 2400 python tools/cpu_model_check.py c2 > gpurun_out/r02d/cpu_model_check_c2.log 2>&1; echo "cpu_model_check rc=$?"
tail -1 gpurun_out/r02d/cpu_model_check_c2.log
timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02d/ref_c3.json 2> gpurun_out/r02d/ref_c3.err; echo "ref rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02d/ref_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['cpu_phases_s'])"
cp .bench_cache/*.json gpurun_out/r02d/ 2>/dev/null
timeout 1500 python bench.py --steps 1 --warmup 1 > gpurun_out/r02d/bench_c3.json 2> gpurun_out/r02d/bench_c3.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/r02d/bench_c3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['solve']['ledger_seconds'], d['cpu_baseline']['value'])"
