# ncu --set full of the temporally blocked 2D elasticity kernel (C3)
cd $GRAFT_REPO_ROOT
CMD="python bench.py --config C3 --steps 1 --warmup 1 --no-cpu --no-e2e --no-kernel-timing"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_elastic2d_tb -c 1 -o gpurun_out/tb_c3 $CMD > gpurun_out/tb_c3.log 2>&1
tail -3 gpurun_out/tb_c3.log
