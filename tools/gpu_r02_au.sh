set -x
T=r02au
for i in 1 2; do
for lean in 1 0; do
  QFB_FWD_LEAN=$lean timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_lean${lean}_$i.json 2>&1
done
done
python tools/show_bench.py gpurun_out/${T}_bench_*.json
