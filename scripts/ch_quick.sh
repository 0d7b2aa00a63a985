#!/bin/bash
# conv_h experiment: role timings, bench, dense-pass parity
TAG=${1:-c}
mkdir -p gpurun_out
CSC_CH_TIMING=1 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cht_${TAG}.log 2>&1
grep conv_h gpurun_out/bench_cht_${TAG}.log | head -1 > gpurun_out/cht_${TAG}.txt
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_ch_${TAG}.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "residual or trajectory_tiny or filter_step" > gpurun_out/pytest_ch_${TAG}.log 2>&1
tail -1 gpurun_out/pytest_ch_${TAG}.log >> gpurun_out/cht_${TAG}.txt
