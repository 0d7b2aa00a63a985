#!/bin/bash
# bench lines for the other BASELINE.json configurations and the p sweep of config 3
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in 0.05 0.2 0.5 1.0; do
  timeout 300 python bench.py --steps 20 --warmup 5 --p $p --no-cpu-baseline > gpurun_out/bench_sweep_p$p.json 2>&1
done
timeout 300 python bench.py --steps 20 --warmup 5 --config batch --no-cpu-baseline > gpurun_out/bench_batch.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --config tiny --no-cpu-baseline > gpurun_out/bench_tiny.json 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --config online --no-cpu-baseline > gpurun_out/bench_online.json 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --config large > gpurun_out/bench_large.json 2>&1
