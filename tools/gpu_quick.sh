# one tiny fused-kernel parity check per variant under a short timeout (deadlock guard)
cd $GRAFT_REPO_ROOT
for v in paper_2509_06971_b200/lib/variants/*.so; do
  echo "== $v"
  PETTO_B200_LIB=$v timeout 25 python -c "import __graft_entry__ as g; g.smoke()" > /tmp/q.log 2>&1
  echo "rc=$?"; tail -2 /tmp/q.log
done
