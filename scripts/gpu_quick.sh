#!/bin/bash
# quick GPU iteration: build, a pytest selection, optional bench (each under its own timeout)
TAG=${1:-q}; shift
SEL=${1:-}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1; echo "build rc=$?" >> gpurun_out/build_${TAG}.log
if [ -n "$SEL" ]; then
  timeout ${PYT_TIMEOUT:-600} python -m pytest tests -m gpu -x -q -k "$SEL" > gpurun_out/pytest_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
fi
if [ -n "${BENCH:-}" ]; then
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
fi
