#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in 1 2 4; do
  CSC_WG_CPT=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/wgb_$c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/wgb_$c.json').readline()); print('cpt=$c', d['value'], d['kernel_rooflines']['wgrad']['avg_launch_ms'])" >> gpurun_out/wg_bench.txt 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_wg2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_wg2.log
