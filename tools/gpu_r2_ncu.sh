#!/bin/bash
# ncu evidence of round 2 (cfg4, one find_solve call of 4 energy points): the launch list (device time
# per launch) and --set full captures of the top kernels in a top-level group (50) and a deep
# contact-row group (242).  Outputs kept small (gpurun_out/ brings back <= 64 MiB): CSV exports, gzip.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
full() {  # name, regex, skip, count, groups...
  local name=$1 rx=$2 sk=$3 cn=$4; shift 4
  timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base mangled \
    -k regex:"$rx" -s $sk -c $cn -o /tmp/n_full_$name -f python tools/run_group.py --config 4 --energies 4 --groups "$@" --profile-groups \
    > gpurun_out/n_ncu_f_$name.log 2>&1
  echo "full $name rc=$?" >> gpurun_out/n_ncu_f.log
  ncu -i /tmp/n_full_$name.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/n_full_$name.raw.csv.gz
  ncu -i /tmp/n_full_$name.ncu-rep --page details 2>/dev/null | gzip > gpurun_out/n_full_$name.details.txt.gz
}
timeout 300 python tools/run_group.py --config 4 --energies 4 --groups 50 242 > gpurun_out/n_rg.log 2>&1 || exit 1
full trail50 'tile_tma_kernelILi4E' 20 2 50
full str50 'tile_tma_kernelILi(8|9|11)E' 0 3 50
full lat50 'panel_cluster_reg|xsolve_kernel|trsm_kernel|gather_kernel' 8 8 50
full tall242 'panel_tall|trsm_kernel|tile_tma_kernelILi4E|panel_inv' 12 8 242
cat gpurun_out/n_ncu_f.log
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file /tmp/n_launches_cfg4.csv python tools/run_group.py --config 4 --energies 4 > gpurun_out/n_ncu_l.log 2>&1
echo "launch list rc=$?" >> gpurun_out/n_ncu_l.log
gzip -c /tmp/n_launches_cfg4.csv > gpurun_out/n_launches_cfg4.csv.gz
tail -2 gpurun_out/n_ncu_l.log; du -sh gpurun_out; ls -la gpurun_out | grep " n_"
