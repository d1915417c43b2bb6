# A/B of kernel variants on the C5 bench (one GPU)
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*.so; do
  echo "== $v" >> gpurun_out/ab.log
  PETTO_B200_LIB=$v timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu 2>&1 | python -c "import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'])
    else: print(l.strip()[:200])" >> gpurun_out/ab.log
done
PETTO_B200_LIB=paper_2509_06971_b200/lib/variants/libpetto_w11.so timeout 900 python -m pytest tests/test_gpu_state.py -x -q -m gpu > gpurun_out/ab_pytest_w11.log 2>&1
tail -3 gpurun_out/ab_pytest_w11.log >> gpurun_out/ab.log
cat gpurun_out/ab.log
