set -x
T=r02ad
for dt in f32 f16; do
  timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_FUSED_FIN=0 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_fused.json 2>&1
cat gpurun_out/${T}_bwd_only.jsonl
python tools/show_bench.py gpurun_out/${T}_bench_*.json
