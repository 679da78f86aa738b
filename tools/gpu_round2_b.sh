#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
FIND_B200_RSYM_DOWN=1 timeout 300 python tools/sym_group_probe.py 32 128 27 > gpurun_out/b_symgroup.log 2>&1
timeout 300 ./tools/dmma_bench > gpurun_out/b_dmma_bench.log 2>&1
timeout 1200 python -m pytest tests/test_fullscale.py -m gpu -x -q -s > gpurun_out/b_fullscale.log 2>&1
