#!/bin/bash
# re-entry call: GPU tests, smoke, cfg4 bench with the driver's default arguments, reference arm
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv > gpurun_out/h_gpu.txt 2>&1
nproc >> gpurun_out/h_gpu.txt; free -g >> gpurun_out/h_gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1
SECONDS=0; timeout 1800 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo "bench rc=$? wall $SECONDS s" >> gpurun_out/h_bench.err
SECONDS=0; timeout 900 python bench.py --impl reference > gpurun_out/h_bench_ref.json 2> gpurun_out/h_bench_ref.err; echo "ref rc=$? wall $SECONDS s" >> gpurun_out/h_bench_ref.err
tail -c 600 gpurun_out/h_pytest.log; tail -c 1500 gpurun_out/h_bench.json
