#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
o=gpurun_out/v_sched.txt; : > $o
run() { echo "== $*" >> $o; env "$@" timeout 600 python tools/step_time.py --config 4 --energies 4 --reps 2 >> $o 2>&1; }
run X=1
run FIND_B200_TMA_SMS=132
run FIND_B200_TMA_SMS=116
run FIND_B200_LANES=2
run FIND_B200_LANES=8
run FIND_B200_PRIO=0
run FIND_B200_GRAPH=0
cat $o
