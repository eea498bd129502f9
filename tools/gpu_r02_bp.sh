# forward tail evict_last (QFB_L2_HINTS=16) with the reversed backward
set -x
T=r02bp
O=gpurun_out
for rep in 1 2 3; do
for h in 0 16 24; do
  QFB_L2_HINTS=$h timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_h${h}_$rep.json 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
