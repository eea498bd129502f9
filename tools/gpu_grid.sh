# Grid over (variant, ring KB) for f32/f16. Outputs -> gpurun_out/grid_*.json
for v in ${VARIANTS:-0}; do for kb in ${RINGS:-72}; do for dt in ${DTYPES:-f32}; do
  QFB_BWD_VARIANT=$v QFB_BWD_RING_KB=$kb timeout 200 python bench.py --no-cpu --no-e2e --no-secondary --steps 300 --dtype $dt > gpurun_out/grid_v${v}_r${kb}_${dt}.json 2>/dev/null
done; done; done
python tools/show_bench.py gpurun_out/grid_*.json
