# temporally blocked 2D heat solve: parity tests and the C2 bench against the per-step-barrier solve
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_state.py tests/test_gpu_acceptance.py tests/test_gpu_design.py -q -m gpu -x 2>&1 | tail -3
for nt in 0 1; do
  PETTO_NO_TBLOCK=$nt timeout 200 python bench.py --config C2 --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('NO_TBLOCK=$nt C2', round(d['value'],2), d['unit'], 'ms/step', round(d['ms_per_step'],4), d['roofline']['kernel'])"
done
