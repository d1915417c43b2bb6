# blocked 2D solves: parity tests, then C1 / C2 / C3
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_state.py -q -m gpu -x -k "temporal" 2>&1 | tail -3
[ -n "$FULL" ] && timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
for c in C1 C2 C3; do
  timeout 200 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('$c', round(d['value'],2), d['unit'], 'ms/step', round(d['ms_per_step'],4), d['roofline']['kernel'])"
done
