#!/bin/bash
TAG=${1:-a}
grep -E "passed|failed|Error|assert|rc=" gpurun_out/pytest_admm_${TAG}.log | head
grep "rel err" gpurun_out/pytest_admm_${TAG}.log | awk '{print $NF}' | sort -g | tail -1
python -c "
import json
l=[x for x in open('gpurun_out/bench_admm_${TAG}.log') if x.startswith('{')][-1]
j=json.loads(l); print(j['value'], j['ms_per_step'])"
python scripts/launch_summary.py gpurun_out/admm_launches_${TAG}.csv | head -${2:-12}
