# C1 K1 time against the tile height (SSTAT_K1_TILE_ROWS); profiles/r02_c1_tile_sweep.log
for tr in 256 512 768 1024 1376 1696 2048 4096; do
  echo "TR=$tr $(SSTAT_K1_TILE_ROWS=$tr python tools/step_time.py 200 2>&1 | grep C1 | tr '\n' ' ')"
done
