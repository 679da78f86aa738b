#!/bin/bash
# A/B of the TMA engine on the Schur / T / R launches (FIND_B200_TMA_MIN_S=0: every group) vs trail only
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
FIND_B200_TMA_MIN_S=0 timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t_pytest_tma_all.log 2>&1; echo "rc=$?" >> gpurun_out/t_pytest_tma_all.log
for cfg in 4 1; do
  ne=4; [ $cfg = 1 ] && ne=16
  FIND_B200_TMA_MIN_S=0 timeout 600 python tools/group_kinds.py --config $cfg --energies $ne --out gpurun_out/t_gk${cfg}_all.json > gpurun_out/t_gk${cfg}_all.txt 2>&1
  timeout 600 python tools/group_kinds.py --config $cfg --energies $ne --out gpurun_out/t_gk${cfg}_def.json > gpurun_out/t_gk${cfg}_def.txt 2>&1
done
tail -3 gpurun_out/t_pytest_tma_all.log
head -3 gpurun_out/t_gk4_all.txt gpurun_out/t_gk4_def.txt gpurun_out/t_gk1_all.txt gpurun_out/t_gk1_def.txt
