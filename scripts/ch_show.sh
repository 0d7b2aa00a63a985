#!/bin/bash
TAG=${1:-c}
cat gpurun_out/cht_${TAG}.txt
python -c "
import json
l=[x for x in open('gpurun_out/bench_ch_${TAG}.log') if x.startswith('{')][-1]
j=json.loads(l); print(j['value'], j['ms_per_step'], {k:round(v['ms_per_step'],3) for k,v in j['kernels'].items()})"
