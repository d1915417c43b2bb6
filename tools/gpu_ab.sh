# A/B of kernel variants: smoke under a tight timeout (deadlock guard), quick
# parity tests, then the C5 bench (one GPU)
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*.so; do
  echo "== $v" >> gpurun_out/ab.log
  PETTO_B200_LIB=$v timeout 40 python -c "import __graft_entry__ as g; g.smoke()" > /tmp/q.log 2>&1
  rc=$?; tail -2 /tmp/q.log >> gpurun_out/ab.log
  if [ $rc -ne 0 ]; then echo "smoke rc=$rc (skipping)" >> gpurun_out/ab.log; continue; fi
  PETTO_B200_LIB=$v timeout 120 python -m pytest tests/test_gpu_state.py -x -q -m gpu -k "elasticity or hybrid" 2>&1 | tail -1 >> gpurun_out/ab.log
  PETTO_B200_LIB=$v timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('GLUPS %.2f  ms/launch %.4f  frac %.3f  clocks %s' % (d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['clocks']))
    else: print(l.strip()[:200])" >> gpurun_out/ab.log
done
cat gpurun_out/ab.log
