#!/bin/bash
# ADMM iteration check: parity tests, a short admm bench, and the launch list
TAG=${1:-a}
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_admm.py -m gpu -q -s -x > gpurun_out/pytest_admm_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/pytest_admm_${TAG}.log
timeout 300 python bench.py --code-solver admm --steps 3 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_admm_${TAG}.log 2>&1; echo rc=$? >> gpurun_out/bench_admm_${TAG}.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/admm_launches_${TAG}.csv python bench.py --code-solver admm --steps 1 --warmup 0 --no-cpu-baseline ${BENCH_ARGS:-} > /dev/null 2>&1
