#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
CSC_TC_DEBUG=8 timeout 300 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2> gpurun_out/tcwait.txt > gpurun_out/tcwait.json
