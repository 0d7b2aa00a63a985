#!/bin/bash
# full ncu capture of the given kernels (one launch each) under the bench command; plain run first
TAG=${1:-x}; shift
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline ${BENCH_ARGS:-}"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 || { echo "plain run failed" >> gpurun_out/ncu_plain_${TAG}.log; exit 1; }
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${TAG}_$k $CMD > gpurun_out/ncu_full_${TAG}_$k.log 2>&1
done
