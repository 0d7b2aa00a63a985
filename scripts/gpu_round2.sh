#!/bin/bash
# round-2 measurement record: parity (all GPU tests incl. the slow config-5 one), smoke, bench on every
# BASELINE.json configuration, the p sweep, the reference arm, the ncu launch list and full captures.
# usage: bash scripts/gpu_round2.sh TAG
TAG=${1:-r02}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
(nproc; lscpu | head -20) > $O/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build rc=$?" >> $O/build.log
timeout -s KILL 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout -s KILL 1800 python -m pytest tests -m gpu -q -s > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
B="timeout -s KILL 600 python bench.py"
$B --steps 20 --warmup 5 > $O/bench_default.log 2>&1
$B --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2>&1
for p in 0.05 0.2 0.5 1.0; do $B --steps 20 --warmup 5 --p $p --no-cpu-baseline > $O/bench_p$p.log 2>&1; done
$B --config batch --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_batch.log 2>&1
$B --config tiny --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_tiny.log 2>&1
$B --config online --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_online.log 2>&1
$B --config large --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_large.log 2>&1
# launch list of the default bench command (ncu after the plain run above exited 0)
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 150 -c 120 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > $O/ncu_launches.log 2>&1
# one full iteration's launches (the iteration boundary: the Lipschitz kernels open each code step)
python scripts/launch_summary.py $O/launches.csv > $O/launches.txt 2>&1
python scripts/trace_run.py --config sweep --iters 100 --out $O/trace_sweep.csv > $O/trace.log 2>&1
bash scripts/ncu_one.sh $TAG code_h conv_h wgrad_h
# the NEXT rows, each on the configuration DESIGN.md §9-§12 quotes
$B --config batch --code-solver admm --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_admm_batch.log 2>&1
$B --config sweep --code-solver admm --steps 3 --warmup 1 --no-cpu-baseline > $O/bench_admm_sweep.log 2>&1
$B --config batch --filter-solver bcd --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_bcd_batch.log 2>&1
$B --config online --filter-solver surrogate --steps 5 --warmup 2 --no-cpu-baseline > $O/bench_surrogate_online.log 2>&1
$B --step-rule eso --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_eso.log 2>&1
