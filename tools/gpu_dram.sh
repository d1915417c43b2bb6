# DRAM bytes + duration of one fused launch per variant (ncu, 3 metrics)
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 1 --warmup 1 --n-apt 3 --no-e2e --no-cpu"
for v in paper_2509_06971_b200/lib/variants/*${1:-}*.so; do
  n=$(basename $v .so)
  PETTO_B200_LIB=$v timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none -k regex:k_elastic3d -s 2 -c 1 --csv $CMD 2>/dev/null | grep -E '"(gpu__time|dram__|lts__)' | awk -F'","' -v n=$n '{print n, $(NF-2), $NF}'
done
