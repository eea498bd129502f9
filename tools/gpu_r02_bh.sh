# L2 eviction hints A/B (QFB_L2_HINTS: 1 fwd x evict_last, 2 bwd x evict_last, 4 bwd up evict_first, 8 bwd dx evict_first)
set -x
T=r02bh
O=gpurun_out
for rep in 1 2; do
for h in 0 1 3 7 15 12 9; do
  QFB_L2_HINTS=$h timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_h${h}_$rep.json 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
