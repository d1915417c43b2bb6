# XD investigation: DRAM bytes per variant, bench of the probe, full captures of base and xd
cd $GRAFT_REPO_ROOT
bash tools/gpu_dram.sh > gpurun_out/xd_dram.log 2>&1
bash tools/gpu_bench_variants.sh xdns > gpurun_out/xd_bench.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --n-apt 3 --no-e2e --no-cpu"
for n in base xd; do
  PETTO_B200_LIB=paper_2509_06971_b200/lib/variants/libpetto_$n.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_elastic3d -s 2 -c 1 -o gpurun_out/prof_$n $CMD > gpurun_out/prof_$n.log 2>&1
done
cat gpurun_out/xd_dram.log gpurun_out/xd_bench.log
