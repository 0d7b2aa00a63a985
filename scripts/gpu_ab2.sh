#!/bin/bash
# Side-by-side timing of several builds of the library on one box, alternating (2 rounds).
# usage: LIBS="ab/libcsc_a.so ab/libcsc_b.so:CSC_X=1" [ARGS="--config sweep"] bash scripts/gpu_ab2.sh
# (an entry lib.so:VAR=VAL runs that build with the environment variable set)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
out=gpurun_out/ab.txt; : > $out
for rep in 1 2; do
  for ent in $LIBS; do
    lib=${ent%%:*}; envv=""; [ "$ent" != "$lib" ] && envv=${ent#*:}
    env $envv CSC_LIB_PATH=$lib timeout -s KILL 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline $ARGS > gpurun_out/ab_run.log 2>&1
    python - "$(basename $lib .so)${envv:+:$envv}" >> $out <<'PY'
import json, sys
l = [x for x in open("gpurun_out/ab_run.log") if x.startswith("{")]
if not l:
    print(sys.argv[1], "FAILED", open("gpurun_out/ab_run.log").read()[-400:]); sys.exit()
j = json.loads(l[-1]); kr = j.get("kernel_rooflines", {})
print(f"{sys.argv[1]:>18} {j['value']:9.2f} it/s  {j['ms_per_step']:.4f} ms  " +
      "  ".join(f"{k} {v.get('avg_launch_ms', 0):.4f}" for k, v in kr.items()) + f"  clk {j['clocks']['sm_mhz']}")
PY
  done
done
cat $out
