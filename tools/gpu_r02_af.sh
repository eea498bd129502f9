set -x
T=r02af
for i in 1 2; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_base_$i.json 2>&1
  QFB_FWD_EXTRA_FLAGS=2 timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_stream_$i.json 2>&1
done
QFB_FWD_EXTRA_FLAGS=2 timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_stream.json 2>&1
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_base.json 2>&1
C5_REPS=40 timeout 120 python tools/c5_probe.py 8 > gpurun_out/${T}_c5.jsonl 2>&1
QFB_FWD_EXTRA_FLAGS=2 C5_REPS=40 timeout 120 python tools/c5_probe.py 8 >> gpurun_out/${T}_c5.jsonl 2>&1
cat gpurun_out/${T}_c5.jsonl
python tools/show_bench.py gpurun_out/${T}_bench_*.json
