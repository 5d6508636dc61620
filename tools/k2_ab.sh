# K2 A/B: this tree vs another package tree (TREE, default the round-1 tree ab/r1), twice each
for i in 1 2; do
  for tree in . ${TREE:-ab/r1}; do
    echo "== $tree"; SWEEP_P=${WIDTHS:-256,136,192,512,1024} timeout 900 python tools/ab/p_sweep_tree.py $tree ${BYTES:-5e10} 2>&1
  done
done
