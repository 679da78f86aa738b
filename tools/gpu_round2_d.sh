#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 120 ./tools/dmma_accuracy > gpurun_out/d_accuracy.log 2>&1
timeout 300 ./tools/dmma_bench > gpurun_out/d_dmma_bench.log 2>&1
