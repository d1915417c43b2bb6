cd $GRAFT_REPO_ROOT
rm -f gpurun_out/bv.log
bash tools/gpu_bench_variants.sh
mkdir -p /tmp/hide; mv paper_2509_06971_b200/lib/variants/libpetto_x*.so /tmp/hide/
bash tools/gpu_prof_ab.sh
