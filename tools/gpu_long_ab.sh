# sustained (power-capped) A/B: the default 10-step bench per variant, no parity gating
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*.so; do
  echo "== $v"
  PETTO_B200_LIB=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('GLUPS %.2f  ms/launch %.4f  clocks %s' % (d['value'], d['roofline']['avg_launch_ms'], d['clocks']))"
done
