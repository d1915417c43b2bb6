# Development runs on one B200: gpurun -- 'bash tools/gpu.sh <what> [TAG]'; logs in gpurun_out/.
#   tests   GPU test suite + smoke()
#   bench   default bench line (CPU baseline + e2e), the reference arm, every BASELINE config
#   prof    ncu launch list + one --set full capture of the fused 3D kernel (C5)
#   slab    compute-side strong scaling of one rank's slab (tools/slab_eff.py, both layouts)
#   loop    device run() loop phase timing at C4 / C5 (tools/run_loop_time.py)
#   ab      per kernel variant in lib/variants/ (tools/build_variants.py): smoke under a
#           deadlock guard, quick parity tests, a 5-step C5 bench
#   cycles  per variant: duration, SM cycles, FP64 / issue utilisation, DRAM bytes (ncu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
WHAT=${1:-tests}
TAG=${2:-run}
O=gpurun_out/${TAG}
case $WHAT in
tests)
  timeout 1800 python -m pytest tests/ -q -m gpu -rf > ${O}_gpu_suite.log 2>&1
  timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${O}_smoke.log 2>&1
  tail -3 ${O}_gpu_suite.log; tail -2 ${O}_smoke.log ;;
bench)
  nproc > ${O}_nproc.txt; lscpu | head -20 >> ${O}_nproc.txt
  timeout 1200 python bench.py > ${O}_bench.json 2> ${O}_bench.err
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_bench_ref.json 2> ${O}_bench_ref.err
  for c in C1 C2 C3 C4; do
    timeout 600 python bench.py --config $c > ${O}_bench_$c.json 2>> ${O}_bench_configs.err
    timeout 600 python bench.py --config $c --impl reference --steps 3 --warmup 1 > ${O}_bench_ref_$c.json 2>> ${O}_bench_configs.err
  done
  cat ${O}_bench.json ${O}_bench_ref.json ;;
prof)
  CMD="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
  $CMD > ${O}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_launches.csv $CMD > ${O}_ncu_list.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elastic3d_fast -s 5 -c 1 -o ${O}_prof $CMD > ${O}_ncu_full.log 2>&1
  tail -2 ${O}_ncu_full.log ;;
slab)
  timeout 900 python tools/slab_eff.py z x > ${O}_slab_eff.log 2>&1; cat ${O}_slab_eff.log ;;
loop)
  for c in C4 C5; do timeout 900 python tools/run_loop_time.py $c $([ $c = C4 ] && echo 20 || echo 3) --x; done > ${O}_loop.log 2>&1
  cat ${O}_loop.log ;;
ab)
  for v in paper_2509_06971_b200/lib/variants/*.so; do
    echo "== $v"
    PETTO_B200_LIB=$v timeout 40 python -c "import __graft_entry__ as g; g.smoke()" > /tmp/q.log 2>&1
    rc=$?; tail -2 /tmp/q.log
    if [ $rc -ne 0 ]; then echo "smoke rc=$rc (skipping)"; continue; fi
    PETTO_B200_LIB=$v timeout 120 python -m pytest tests/test_gpu_state.py -x -q -m gpu -k "elasticity or hybrid" 2>&1 | tail -1
    PETTO_B200_LIB=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | grep '^{'
  done > ${O}_ab.log 2>&1; cat ${O}_ab.log ;;
cycles)
  CMD="python bench.py --steps 1 --warmup 1 --n-apt 4 --no-e2e --no-cpu"
  M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
  for v in paper_2509_06971_b200/lib/variants/*${3:-}*.so; do
    n=$(basename $v .so); n=${n#libpetto_}
    PETTO_B200_LIB=$v timeout 300 ncu --metrics $M --clock-control none -k regex:k_elastic3d -s 2 -c 3 --csv $CMD 2>/dev/null \
      | grep -E '"(gpu__|sm__|smsp__|dram__)' | awk -F'","' -v n=$n '{gsub(/"/,"",$NF); print n, $(NF-2), $NF}'
  done > ${O}_cycles.log; cat ${O}_cycles.log ;;
*) echo "unknown: $WHAT"; exit 2 ;;
esac
