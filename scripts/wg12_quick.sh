#!/bin/bash
# filter-gradient converter-count experiment: bench + filter-step parity
mkdir -p gpurun_out
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_wg12.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_wg12.log').readline()); print(d['value'], d['kernel_rooflines']['wgrad']['avg_launch_ms'])" > gpurun_out/wg12.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "filter_step or trajectory or wgrad" > gpurun_out/pytest_wg12.log 2>&1
tail -1 gpurun_out/pytest_wg12.log >> gpurun_out/wg12.txt
