# slot-probe variants (tools/cta_times.py) -- probe builds, results wrong by construction
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*${1:-slots}*.so; do
  echo "== $v"; PETTO_B200_LIB=$v timeout 300 python tools/cta_times.py 2>&1 | grep -E "kernel span|slots|first owned"
done
