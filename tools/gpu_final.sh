# round-end validation: GPU suite, smoke, default bench + reference arm, launch list, full capture
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
bash tools/gpu_bench_full.sh ${1:-r01c}
