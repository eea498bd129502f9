# consumer-layout A/B: parity of every layout, backward alone and in the step
set -x
T=r02s
timeout 900 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for dt in f32 f16; do
  for impl in tile8 tile8m quad quadm; do
    QFB_BWD_IMPL=$impl timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
  QFB_BWD_IMPL=quadm QFB_BWD_VARIANT=360 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_IMPL=quadm QFB_BWD_VARIANT=368 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_VARIANT=8 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_VARIANT=16 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
for impl in tile8 quadm; do
  for dt in f32 f16; do
    QFB_BWD_IMPL=$impl timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype $dt > gpurun_out/${T}_bench_${dt}_${impl}.json 2>&1
  done
done
cat gpurun_out/${T}_bwd_only.jsonl
