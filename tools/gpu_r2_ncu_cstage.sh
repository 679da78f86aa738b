#!/bin/bash
# --set full captures of trailing-update launches with and without the staged C block (groups 242 and 50)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for cs in 0 1; do
  FIND_B200_CSTAGE=$cs timeout 300 python tools/run_group.py --config 4 --energies 4 --groups 242 50 > gpurun_out/nc_rg$cs.log 2>&1 || exit 1
  FIND_B200_CSTAGE=$cs timeout 900 ncu --set full --clock-control none --profile-from-start off --kernel-name-base mangled \
    -k regex:'tile_tma_kernelILi4E' -s 5 -c 6 -o /tmp/nc_full_$cs -f python tools/run_group.py --config 4 --energies 4 --groups 242 50 --profile-groups \
    > gpurun_out/nc_ncu_$cs.log 2>&1
  echo "cs=$cs rc=$?" >> gpurun_out/nc.log
  ncu -i /tmp/nc_full_$cs.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/nc_full_cs$cs.raw.csv.gz
  ncu -i /tmp/nc_full_$cs.ncu-rep --page details 2>/dev/null | gzip > gpurun_out/nc_full_cs$cs.details.txt.gz
done
cat gpurun_out/nc.log; ls -la gpurun_out/nc_*
