# temporally blocked 2D elasticity: parity tests, then C1 / C3 against the per-step-barrier solve
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_state.py -q -m gpu -x -k "elastic2d_temporal or heat2d_temporal" 2>&1 | tail -15
[ -n "$FULL" ] && timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
for c in C1 C3; do
for nt in 0 1; do
  PETTO_NO_TBLOCK=$nt timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('NO_TBLOCK=$nt $c', round(d['value'],2), d['unit'], 'ms/step', round(d['ms_per_step'],4), d['roofline']['kernel'])"
done
done
