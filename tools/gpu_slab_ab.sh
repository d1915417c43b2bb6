# slab-efficiency probe per variant library (tools/slab_eff.py)
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*${1:-}*.so; do
  echo "== $v"; PETTO_B200_LIB=$v STEPS=40 timeout 300 python tools/slab_eff.py 2>&1 | tail -1
done
