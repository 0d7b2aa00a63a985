O=gpurun_out/wh3; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "filter_step" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in 1 2 4; do CSC_WH_CPT=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_cpt$c.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:wgrad_h -s 3 -c 1 -o $O/prof_wgrad_h python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
