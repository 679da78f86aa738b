#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
O=gpurun_out/c_err.jsonl; : > $O
timeout 300 python tools/err_probe.py 1 2 >> $O 2>&1
timeout 300 python tools/err_probe.py 1 2 --sym 0 >> $O 2>&1
FIND_B200_NB=16 timeout 300 python tools/err_probe.py 1 2 >> $O 2>&1
FIND_B200_NB=8 timeout 300 python tools/err_probe.py 1 2 >> $O 2>&1
FIND_B200_STRUCT=0 timeout 300 python tools/err_probe.py 1 2 >> $O 2>&1
FIND_B200_WIDE_MIN_S=100000 timeout 300 python tools/err_probe.py 1 2 >> $O 2>&1
FIND_B200_SMEM_PANEL=1 timeout 300 python tools/err_probe.py 1 >> $O 2>&1
