#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bdbg.log 2>&1
for d in 0 64 128 192 65 193; do
  CSC_TC_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dbg_$d.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/dbg_$d.log').readline()); print('dbg=$d', d['kernel_rooflines']['conv']['avg_launch_ms'])" >> gpurun_out/dbg_sweep2.txt 2>&1
done
