#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/i8_probe 256 512 1024
timeout 120 ./tools/i8_probe 384 768 4096
python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py -q -m gpu -k "dist or backup" 2>&1 | tail -3
