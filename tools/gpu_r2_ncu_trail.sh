#!/bin/bash
# DRAM bytes of every trailing-update launch of one cfg4 solve (4 energy points): the per-launch average is
# bench.py's roofline.traffic (ncu serialises and flushes caches: an upper bound of the in-flight traffic)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/run_group.py --config 4 --energies 4 --groups 50 > gpurun_out/nt_rg.log 2>&1 || exit 1
timeout 3000 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --kernel-name-base mangled -k regex:'tile_tma_kernelILi4E' --log-file /tmp/nt_trail.csv \
  python tools/run_group.py --config 4 --energies 4 > gpurun_out/nt_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/nt_ncu.log
gzip -c /tmp/nt_trail.csv > gpurun_out/nt_trail_launches_cfg4.csv.gz
tail -2 gpurun_out/nt_ncu.log; ls -la gpurun_out/nt_*
