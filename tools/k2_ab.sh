# K2 A/B: this tree vs another package tree (TREE: a built copy of the package, e.g. made with
# `git archive <rev> paper_2604_23826_b200 include | tar -x -C ab/<name>` and `make -C
# ab/<name>/paper_2604_23826_b200/csrc`), twice each.  The experiment trees of the round-2 logs
# (ab/nowait, ab/nopre, ...) were such copies with one change each, described in the logs.
: "${TREE:?set TREE to the package tree to compare with}"
for i in 1 2; do
  for tree in . "$TREE"; do
    echo "== $tree"; SWEEP_P=${WIDTHS:-256,136,192,512,1024} timeout 900 python tools/ab/p_sweep_tree.py $tree ${BYTES:-5e10} 2>&1
  done
done
