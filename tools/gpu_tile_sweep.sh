# Memory-only backward probe across tile sizes (tune/libqfb_g*.so builds) and ring budgets.
for lib in tune/libqfb_g7.so paper_2511_12653_b200/libqfb.so tune/libqfb_g9.so; do
  for kb in ${RINGS:-44 72 100 140}; do
    QFB_LIB_PATH=$PWD/$lib QFB_BWD_VARIANT=${V:-8} QFB_BWD_RING_KB=$kb timeout 200 python bench.py --no-cpu --no-e2e --no-secondary --steps 300 > gpurun_out/tile_$(basename $lib .so)_r$kb.json 2>/dev/null
  done
done
python tools/show_bench.py gpurun_out/tile_*.json
