#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_paths.py -m gpu -x -q -k "tall" > gpurun_out/u_pytest_tall.log 2>&1; echo "rc=$?" >> gpurun_out/u_pytest_tall.log
tail -15 gpurun_out/u_pytest_tall.log
timeout 600 python tools/group_kinds.py --config 4 --energies 4 --out gpurun_out/u_gk4_tall.json > gpurun_out/u_gk4_tall.txt 2>&1
FIND_B200_TALL_MIN_PANELS=0 timeout 600 python tools/group_kinds.py --config 4 --energies 4 --out gpurun_out/u_gk4_tall0.json > gpurun_out/u_gk4_tall0.txt 2>&1
FIND_B200_TALL_MIN_PANELS=0 FIND_B200_TALL_MIN_ROWS=96 timeout 600 python tools/group_kinds.py --config 1 --energies 16 --out gpurun_out/u_gk1_tall0.json > gpurun_out/u_gk1_tall0.txt 2>&1
head -3 gpurun_out/u_gk4_tall.txt gpurun_out/u_gk4_tall0.txt gpurun_out/u_gk1_tall0.txt
