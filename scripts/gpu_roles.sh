# per-role cycle counters of the tensor-core kernels (tuning build; not the product build)
O=gpurun_out/${1:-roles}; mkdir -p $O
CSC_NVCC_EXTRA=-DCSC_ROLE_TIMING python -c "from paper_1909_00145_b200 import build as b; b.build(force=True)" > $O/build.log 2>&1
timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-graph > $O/bench_roles.log 2>&1
grep roles $O/bench_roles.log | tail -12
python -c "from paper_1909_00145_b200 import build as b; b.build(force=True)" > $O/build2.log 2>&1
