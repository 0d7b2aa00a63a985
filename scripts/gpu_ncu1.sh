# one full ncu capture of the named kernel under the default bench command (plain run first)
O=gpurun_out/${1:-ncu1}; K=${2:-wgrad_h}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $O/prof_$K python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
