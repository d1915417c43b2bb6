# full ncu capture (one launch, source-correlated) of the fused 3D kernel for
# every variant library; reports land in gpurun_out/prof_<name>.ncu-rep
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --n-apt 3 --no-e2e --no-cpu"
for v in paper_2509_06971_b200/lib/variants/*.so; do
  n=$(basename $v .so); n=${n#libpetto_}
  PETTO_B200_LIB=$v timeout 60 $CMD > /dev/null 2>&1 || { echo "$n: plain run failed"; continue; }
  PETTO_B200_LIB=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_elastic3d -s 2 -c 1 \
     -o gpurun_out/prof_$n $CMD > gpurun_out/prof_$n.log 2>&1
  echo "$n: ncu rc=$?"
done
