# x-split walk of the fused 3D kernel: smoke (deadlock guard), bit-identity tests,
# the 3D parity suites, then C4 / C5 and the N=8 slab compute side
cd $GRAFT_REPO_ROOT
L=gpurun_out/xsplit.log; : > $L
timeout 60 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1 || { echo "smoke failed rc=$?" >> $L; cat $L; exit 1; }
timeout 300 python -m pytest tests/test_gpu_state.py -x -q -m gpu -k "split_walk" 2>&1 | tail -15 >> $L
timeout 900 python -m pytest tests/test_gpu_state.py tests/test_gpu_slab.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py -x -q -m gpu 2>&1 | tail -3 >> $L
for cfg in C4 C5 C4; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$cfg GLUPS %.2f ms/step %.4f ms/launch %.4f clocks %s' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz']))" >> $L
done
for pl in 6,4 10,2 22,1; do PETTO_E3_PLAN=$pl timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>/dev/null | grep -o '"value": [0-9.]*' | sed "s/^/C4 plan $pl: /" >> $L; done
timeout 600 python tools/slab_eff.py >> $L 2>&1
cat $L
