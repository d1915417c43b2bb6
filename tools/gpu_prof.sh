# profile the fused 3D elasticity kernel on C5 (one GPU)
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --n-apt 3 --no-e2e --no-cpu"
timeout 900 python -m pytest tests/test_gpu_state.py -x -q -m gpu > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu > gpurun_out/r2_bench.log 2>&1
$CMD > gpurun_out/r2_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elastic3d -s 2 -c 1 -o gpurun_out/r2_prof_e3 $CMD > gpurun_out/r2_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2_ncu.log
tail -3 gpurun_out/r2_pytest.log; tail -2 gpurun_out/r2_bench.log; tail -3 gpurun_out/r2_ncu.log
