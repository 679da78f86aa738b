#!/bin/bash
# first round-2 GPU call: GPU tests, symmetric-R probe, cfg4 bench with the driver's arguments
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/a_gpu.txt 2>&1
nproc >> gpurun_out/a_gpu.txt; free -g >> gpurun_out/a_gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/a_pytest.log
FIND_B200_RSYM_DOWN=1 timeout 600 python tools/sym_probe.py 64 256 > gpurun_out/a_sym_64x256.log 2>&1
FIND_B200_RSYM_DOWN=1 timeout 600 python tools/sym_probe.py 32 128 > gpurun_out/a_sym_32x128.log 2>&1
SECONDS=0; timeout 1800 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; echo "bench wall $SECONDS s" >> gpurun_out/a_bench.err
echo "bench rc=$?" >> gpurun_out/a_bench.err
