# full bench line (with CPU baseline + e2e), reference arm, ncu launch list and full capture
cd $GRAFT_REPO_ROOT
TAG=${1:-b}
nproc > gpurun_out/${TAG}_nproc.txt; lscpu | head -20 >> gpurun_out/${TAG}_nproc.txt
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_list.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elastic3d -s 3 -c 1 -o gpurun_out/${TAG}_prof_e3 $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu_full.log
cat gpurun_out/${TAG}_bench.json; tail -2 gpurun_out/${TAG}_bench.err; cat gpurun_out/${TAG}_bench_ref.json; tail -2 gpurun_out/${TAG}_ncu_full.log
