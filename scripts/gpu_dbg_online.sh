python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for v in "X=1" "CSC_WGRAD_PATH=tf32" "CSC_WH_CPT=1"; do
  echo "== $v"; env $v timeout 600 python -m pytest tests/test_gpu_trajectories.py -q -x -s -k online 2>&1 | grep -E "AssertionError|online worst|passed|failed" | cut -c1-400
done
