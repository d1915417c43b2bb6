# PDL variant check: wait at kernel entry (no setup overlap); C4/C5 bench, C5 ncu
# instruction count and time, 3D parity subset
cd $GRAFT_REPO_ROOT
L=gpurun_out/pdl2.log; : > $L
timeout 60 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1 || { echo "smoke failed" >> $L; cat $L; exit 1; }
timeout 600 python -m pytest tests/test_gpu_state.py tests/test_gpu_slab.py tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -1 >> $L
for cfg in C4 C5 C4 C5; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$cfg GLUPS %.2f ms/step %.4f ms/launch %.4f clocks %s' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz']))" >> $L
done
CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_elastic3d -s 3 -c 3 --csv $CMD 2>/dev/null | grep -E "k_elastic3d" | cut -c1-40,200-400 | tail -9 >> $L
cat $L
