#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
o=gpurun_out/x_cfg1.txt; : > $o
run() { echo "== $*" >> $o; env "$@" timeout 600 python tools/step_time.py --config 1 --energies 16 --reps 5 >> $o 2>&1; }
run X=1
run FIND_B200_TMA_MIN_S=1000000 
run FIND_B200_TMA_MIN_S=1000000 FIND_B200_TMA_TRAIL_MIN_N=256
run FIND_B200_TMA_MIN_S=128 FIND_B200_TMA_TRAIL_MIN_N=192
run FIND_B200_TMA=0
run FIND_B200_TMA_SMS=64
run FIND_B200_TMA_SMS=32
cat $o
