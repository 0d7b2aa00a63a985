#!/bin/bash
# block-level atomics check: ADMM parity + bench + launch list, hot-path parity subset + bench
TAG=${1:-b}
mkdir -p gpurun_out
bash scripts/admm_quick.sh $TAG
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_eso.py -m gpu -q -x > gpurun_out/pytest_hot_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/pytest_hot_${TAG}.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
