# run the GPU test suite + smoke on one B200; logs under gpurun_out/
cd $GRAFT_REPO_ROOT
TAG=${1:-t}
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
tail -15 gpurun_out/${TAG}_pytest.log; tail -3 gpurun_out/${TAG}_smoke.log
