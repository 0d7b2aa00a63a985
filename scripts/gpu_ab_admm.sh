# which conv_h variant fails the ADMM sweep bench / the online trajectory
for flags in "$@"; do
  CSC_NVCC_EXTRA="$flags" python -c "from paper_1909_00145_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  a=$(timeout 300 python bench.py --config sweep --code-solver admm --steps 2 --warmup 1 --no-cpu-baseline 2>&1 | grep -E 'CSCError|timed region' | tail -1 | cut -c1-120)
  t=$(timeout 600 python -m pytest tests/test_gpu_trajectories.py -q -x -k online 2>&1 | tail -1)
  echo "[$flags] admm: $a | online: $t"
done
python -c "from paper_1909_00145_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
