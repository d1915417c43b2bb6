# A/B of programmatic dependent launch between fused 3D steps (PETTO_NO_PDL=1 = off):
# smoke + 3D parity tests with PDL on, then C4 / C5 bench lines, alternating
cd $GRAFT_REPO_ROOT
L=gpurun_out/pdl_ab.log; : > $L
timeout 60 python -c "import __graft_entry__ as g; g.smoke()" >> $L 2>&1 || { echo "smoke failed" >> $L; cat $L; exit 1; }
timeout 600 python -m pytest tests/test_gpu_state.py tests/test_gpu_fullsize.py tests/test_gpu_acceptance.py -x -q -m gpu 2>&1 | tail -2 >> $L
for rep in 1 2; do
for cfg in C4 C5; do
for pdl in 0 1; do
  PETTO_NO_PDL=$pdl timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu ${EXTRA} 2>/dev/null | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$cfg no_pdl=$pdl GLUPS %.2f ms/step %.4f ms/launch %.4f clocks %s' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz']))" >> $L
done; done; done
for pdl in 0 1; do
  PETTO_NO_PDL=$pdl timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-e2e --no-cpu --no-kernel-timing 2>/dev/null | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('C4 no-kernel-timing no_pdl=$pdl GLUPS %.2f ms/step %.4f' % (d['value'], d['ms_per_step']))" >> $L
done
cat $L
