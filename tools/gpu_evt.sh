# effect of the per-launch timing events on the measured step (C5 and C4)
cd $GRAFT_REPO_ROOT
for c in C5 C4; do for i in 1 2; do for kt in "" "--no-kernel-timing"; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e $kt 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('$c', '${kt:-events}', round(d['value'],2), 'ms/step', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'])"
done; done; done
