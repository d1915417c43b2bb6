# Per variant: duration, SM cycles (clock-independent) and FP64/issue utilisation
# of three fused launches under ncu; one GPU.  Optional arg: variant name pattern.
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --n-apt 4 --no-e2e --no-cpu"
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
for v in paper_2509_06971_b200/lib/variants/*${1:-}*.so; do
  n=$(basename $v .so); n=${n#libpetto_}
  PETTO_B200_LIB=$v timeout 300 ncu --metrics $M --clock-control none -k regex:k_elastic3d -s 2 -c 3 --csv $CMD 2>/dev/null \
    | grep -E '"(gpu__|sm__|smsp__|dram__)' | awk -F'","' -v n=$n '{gsub(/"/,"",$NF); print n, $(NF-2), $NF}'
done
