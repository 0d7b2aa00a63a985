#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bw.log 2>&1
for d in 8 63; do
  echo "== dbg=$d" >> gpurun_out/waitprof2.txt
  CSC_TC_DEBUG=$d timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>> gpurun_out/waitprof2.txt > gpurun_out/wp_$d.json
  python -c "import json; d=json.loads(open('gpurun_out/wp_$d.json').readline()); print('ms', d['kernel_rooflines']['conv']['avg_launch_ms'])" >> gpurun_out/waitprof2.txt 2>&1
done
