cd $GRAFT_REPO_ROOT
nvidia-smi -L > gpurun_out/r1_env.log 2>&1
timeout 900 python -m pytest tests/test_gpu_state.py -x -q -m gpu > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu > gpurun_out/r1_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r1_bench.log
tail -5 gpurun_out/r1_pytest.log; tail -3 gpurun_out/r1_smoke.log; tail -3 gpurun_out/r1_bench.log
