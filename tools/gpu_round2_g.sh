#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g_pytest.log
# launch list of one cfg4 solve (4 energy points: one find_solve call of the bench step)
timeout 300 python tools/run_group.py --config 4 --energies 4 > gpurun_out/g_rg.log 2>&1 && \
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/g_launches_cfg4.csv python tools/run_group.py --config 4 --energies 4 > gpurun_out/g_ncu_l.log 2>&1
echo "launch list rc=$?" >> gpurun_out/g_ncu_l.log
# full-set captures of the top kernels in a top-level group (50) and a deep contact group (151)
timeout 1800 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"tile_tma|rgemm_kernel|schur_kernel|xsolve|panel_cluster_reg|trsm_kernel|tgemm_kernel" -c 24 \
  -o gpurun_out/g_full_cfg4 python tools/run_group.py --config 4 --energies 4 --groups 50 151 --profile-groups > gpurun_out/g_ncu_f.log 2>&1
echo "full rc=$?" >> gpurun_out/g_ncu_f.log
