# per-warp cycle accounting (E3_EXPERIMENT=3 build): barrier / full-barrier waits
cd $GRAFT_REPO_ROOT
PETTO_B200_LIB=paper_2509_06971_b200/lib/variants/libpetto_x3.so timeout 120 python bench.py --steps 1 --warmup 1 --n-apt 3 --no-e2e --no-cpu > gpurun_out/x3.log 2>&1
grep prof gpurun_out/x3.log | sort -k3n -k5n | head -40
