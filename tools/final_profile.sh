# Round-end evidence refresh (one GPU call): smoke(), bench line, all-config table, ncu launch list
# of one cfg1 solve and an ncu --set full capture of the first rgemm / trail / panel launches after 60.
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 1800 python tools/config_table.py --configs 0,1,2,3,4 --offdiag3 2>&1 | grep "^{" > gpurun_out/config_table_final.jsonl
python tools/run_group.py && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv python tools/run_group.py > gpurun_out/ncu_l.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"rgemm|trail|panel1" -s 60 -c 6 -o gpurun_out/full_final python tools/run_group.py > gpurun_out/ncu_f.log 2>&1
tail -c 300 gpurun_out/bench_final.json; wc -l gpurun_out/config_table_final.jsonl
