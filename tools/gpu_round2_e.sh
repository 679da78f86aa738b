#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e_pytest.log
timeout 600 python -m pytest tests/test_fullscale.py -m gpu -q -s > gpurun_out/e_fullscale.log 2>&1
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/e_bench1_tma.json 2> gpurun_out/e_bench1_tma.err
FIND_B200_TMA=0 timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/e_bench1_old.json 2> gpurun_out/e_bench1_old.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1 > gpurun_out/e_bench4_tma.json 2> gpurun_out/e_bench4_tma.err
