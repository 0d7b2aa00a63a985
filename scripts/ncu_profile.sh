#!/bin/bash
# ncu evidence for the bench workload: launch list (cold-cache, serialised) and full captures of the
# top kernels.  Usage: bash scripts/ncu_profile.sh <tag> [kernel regex ...]
TAG=${1:-r01}; shift
KERNELS=${@:-conv_fwd wgrad_kernel code_step}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ncu_build.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain_${TAG}.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
for k in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${TAG}_$k $CMD > gpurun_out/ncu_full_${TAG}_$k.log 2>&1
done
ls -la gpurun_out/
