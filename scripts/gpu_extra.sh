#!/bin/bash
# extra evidence at one commit: e2e vs steps (fixed or per-step overhead), the ADMM solver over p, one ncu
# source-level capture of the dense pass (shared-memory bank conflicts per instruction)
O=gpurun_out/${1:-extra}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for K in 20 100 400; do
  timeout 300 python bench.py --steps $K --warmup 3 --no-cpu-baseline > $O/bench_steps$K.json 2> $O/bench_steps$K.err
done
for P in 0.02 0.05 0.1 0.2 0.5; do
  timeout 300 python bench.py --config batch --code-solver admm --p $P --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_admm_batch_p$P.json 2> $O/bench_admm_batch_p$P.err
done
for P in 0.02 0.1 0.5; do
  timeout 300 python bench.py --code-solver admm --p $P --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_admm_sweep_p$P.json 2> $O/bench_admm_sweep_p$P.err
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_h_kernel -s 3 -c 1 -o $O/prof_conv_h python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
ls -la $O
