# full GPU suite, every BASELINE config with its CPU baseline, and ncu of the blocked 2D kernels
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
bash tools/gpu_configs.sh
for c in C1:elastic2d C3:elastic2d C2:heat2d; do
  cfg=${c%%:*}; k=${c##*:}
  CMD="python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu --no-e2e --no-kernel-timing"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_${k}_tb -c 1 -o gpurun_out/tb_$cfg $CMD > gpurun_out/tb_$cfg.log 2>&1
done
ls gpurun_out/tb_*
