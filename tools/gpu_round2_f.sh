#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/f_pytest.log
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra --e2e-steps 1"
FIND_B200_TMA_MIN_S=0 FIND_B200_TMA_TRAIL_MIN_N=0 timeout 900 $B --config 4 --levels gpurun_out/f_lv4_all.json > gpurun_out/f_b4_all.json 2>gpurun_out/f_b4_all.err
FIND_B200_TMA=0 timeout 900 $B --config 4 --levels gpurun_out/f_lv4_none.json > gpurun_out/f_b4_none.json 2>gpurun_out/f_b4_none.err
FIND_B200_TMA_MIN_S=0 FIND_B200_TMA_TRAIL_MIN_N=0 timeout 600 $B --config 1 --levels gpurun_out/f_lv1_all.json > gpurun_out/f_b1_all.json 2>gpurun_out/f_b1_all.err
FIND_B200_TMA=0 timeout 600 $B --config 1 --levels gpurun_out/f_lv1_none.json > gpurun_out/f_b1_none.json 2>gpurun_out/f_b1_none.err
FIND_B200_RSYM_DOWN=1 timeout 600 python tools/sym_prefix_probe.py 64 256 > gpurun_out/f_symprefix.log 2>&1
