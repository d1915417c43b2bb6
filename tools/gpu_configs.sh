# every BASELINE config: device GLUPS (bench.py --config Cx) beside the reference's CPU path
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/cfg_nproc.txt
for spec in C1:500 C2:500 C3:100 C4:20; do
  c=${spec%%:*}; n=${spec##*:}
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --cpu-steps $n > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  python -c "import json; d=json.load(open('gpurun_out/cfg_$c.json')); cb=d.get('cpu_baseline',{}); print('$c', d['config']['workload'][:60], '|', round(d['value'],2), d['unit'], '| kernel', d['roofline']['kernel'], '| cpu', round(cb.get('value',0),4), cb.get('cores'), cb.get('kind'), cb.get('sample','')[:50])"
done
CMD="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg_C2_launches.csv $CMD > /dev/null 2>&1
CMD="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg_C3_launches.csv $CMD > /dev/null 2>&1
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu --no-e2e"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg_C4_launches.csv $CMD > /dev/null 2>&1
ls gpurun_out/cfg_*
