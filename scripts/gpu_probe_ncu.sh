#!/bin/bash
timeout -s KILL 300 python scripts/tau_probe.py > gpurun_out/tau_probe.log 2>&1
bash scripts/ncu_one.sh r2a code_h
ncu -i gpurun_out/prof_r2a_code_h.ncu-rep --page raw --csv > gpurun_out/prof_r2a_code_h_raw.csv 2>&1
