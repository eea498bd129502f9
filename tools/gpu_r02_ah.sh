set -x
T=r02ah
for m in 4 5 6 12 13; do
  QFB_PDL=$m timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_pdl$m.json 2>&1
done
python tools/show_bench.py gpurun_out/${T}_bench_*.json
