#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for d in 24 40 56 63; do
echo "== dbg=$d" >> gpurun_out/tcwait2.txt
CSC_TC_DEBUG=$d timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>> gpurun_out/tcwait2.txt > /dev/null
done
