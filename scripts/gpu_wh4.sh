O=gpurun_out/${1:-wh4}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "filter_step" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench.log 2>&1
grep '^{"metric"' $O/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['avg_launch_ms'],4) for k,v in d['kernel_rooflines'].items()})"
bash scripts/gpu_roles.sh ${1:-wh4}_roles
