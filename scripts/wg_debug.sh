#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/wgdbg_build.log 2>&1
for d in 31 30 29 27 23 15 0; do
  echo "== dbg=$d" >> gpurun_out/wgdbg.txt
  CSC_WG_DEBUG=$d timeout 120 python -m pytest tests -m gpu -x -q -k "filter_step_parity and shape0-tc" 2>&1 | grep -E "passed|failed|Error|error" | head -3 >> gpurun_out/wgdbg.txt
done
