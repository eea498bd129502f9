# L2 bulk prefetch in the backward producer: parity + backward alone + step
set -x
T=r02y
timeout 600 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider -k "tiledp or default" > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for dt in f32 f16; do
  for impl in tiled tiledp tiled tiledp; do
    QFB_BWD_IMPL=$impl timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
done
for impl in tiled tiledp; do
  QFB_BWD_IMPL=$impl timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_${impl}.json 2>&1
  QFB_BWD_IMPL=$impl timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_${impl}.json 2>&1
done
cat gpurun_out/${T}_bwd_only.jsonl
python tools/show_bench.py gpurun_out/${T}_bench_*.json
