#!/bin/bash
# A/B GPU check: parity subset, then the bench under each CSC_CH_WAIT mode
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_trajectories.py -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
for m in 0 1; do
  CSC_CH_WAIT=$m timeout -s KILL 300 python bench.py --steps 20 --warmup 3 > gpurun_out/b_w$m.log 2>&1
  echo "bench rc=$?" >> gpurun_out/b_w$m.log
done
