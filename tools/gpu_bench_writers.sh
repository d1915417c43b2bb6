cd $GRAFT_REPO_ROOT
df -h /tmp | tail -1 > gpurun_out/wb_df.txt
timeout 600 python tools/bench_writers.py > gpurun_out/wb.json 2> gpurun_out/wb.err; echo rc=$? >> gpurun_out/wb.err
CMD="python tools/bench_writers.py --nz 32 --sample 100000"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/wb_launches.csv $CMD > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block_write -s 2 -c 1 -o gpurun_out/wb_prof $CMD > gpurun_out/wb_ncu.log 2>&1
cat gpurun_out/wb.json; tail -3 gpurun_out/wb.err; cat gpurun_out/wb_df.txt; tail -1 gpurun_out/wb_ncu.log
