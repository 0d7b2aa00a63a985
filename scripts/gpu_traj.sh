#!/bin/bash
# the 50-iteration trajectory tests (BASELINE configs 2-5)
timeout -s KILL 1500 python -m pytest tests/test_gpu_trajectories.py -x -q -s ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/traj.log 2>&1
echo "rc=$?" >> gpurun_out/traj.log
