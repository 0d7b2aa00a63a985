#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bw.log 2>&1
for d in 8 9 10 14 15; do
  echo "== dbg=$d" >> gpurun_out/waitprof.txt
  CSC_TC_DEBUG=$d timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>> gpurun_out/waitprof.txt > /dev/null
done
