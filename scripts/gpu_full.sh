#!/bin/bash
# build, smoke, GPU parity tests, bench, launch list (ncu), one full capture per requested kernel
TAG=${1:-dev}; shift
KERNELS=${@:-}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi_${TAG}.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1; echo "build rc=$?" >> gpurun_out/build_${TAG}.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_${TAG}.log
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_${TAG}.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_${TAG}.log
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS:-} > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_${TAG}.log
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-}"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
for k in $KERNELS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 6 -c 1 -o gpurun_out/prof_${TAG}_$k $CMD > gpurun_out/ncu_full_${TAG}_$k.log 2>&1
done
ls -la gpurun_out/
