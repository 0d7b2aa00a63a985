#!/bin/bash
# quick GPU check: selected parity tests + a short bench (round 2 iteration loop)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b.log 2>&1
echo "bench rc=$?" >> gpurun_out/b.log
