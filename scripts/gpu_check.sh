#!/bin/bash
# quick check of a kernel change: build, the default bench line, then the GPU suite (PYTEST_K filters it)
O=gpurun_out/${1:-chk}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo "build failed"; tail -20 $O/build.log; exit 1; }
timeout -s KILL 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS:-} > $O/bench_default.log 2>&1; echo "bench rc=$?" >> $O/bench_default.log
tail -2 $O/bench_default.log | cut -c1-600
timeout -s KILL 1200 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
tail -15 $O/pytest_gpu.log
