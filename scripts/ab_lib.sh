# A/B over library variants: LIBS="base var_a var_b" (base = the in-tree build)
cd $GRAFT_REPO_ROOT
L=paper_2305_02522_b200/libbitgnn_b200.so
cp $L build/base.so
for v in ${LIBS:-base}; do
  cp build/$v.so $L
  echo "######## $v"
  [ -n "$TESTS" ] && timeout 900 python -m pytest $TESTS -x -q 2>&1 | tail -2
  ENVS="${ENVS:-}" bash scripts/ab.sh
done
cp build/base.so $L
