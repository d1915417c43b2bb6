# C5 bench of every variant library without parity gating (for experiment
# builds whose results are deliberately wrong); one GPU
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*${1:-}*.so; do
  echo "== $v" >> gpurun_out/bv.log
  PETTO_B200_LIB=$v timeout 120 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('GLUPS %.2f  ms/launch %.4f  frac %.3f  clocks %s' % (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']))
    else: print(l.strip()[:200])" >> gpurun_out/bv.log
done
cat gpurun_out/bv.log
