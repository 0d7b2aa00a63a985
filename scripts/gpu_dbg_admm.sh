python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
echo "tf32: $(CSC_WGRAD_PATH=tf32 timeout 300 python bench.py --config sweep --code-solver admm --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -E 'CSCError|it/s' | tail -1 | cut -c1-200)"
echo "blocking: $(CUDA_LAUNCH_BLOCKING=1 timeout 300 python bench.py --config sweep --code-solver admm --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -E 'CSCError|it/s' | tail -1 | cut -c1-300)"
echo "online traj: $(timeout 600 python -m pytest tests/test_gpu_trajectories.py -q -x -k online 2>&1 | tail -1)"
echo "online traj tf32: $(CSC_WGRAD_PATH=tf32 timeout 600 python -m pytest tests/test_gpu_trajectories.py -q -x -k online 2>&1 | tail -1)"
