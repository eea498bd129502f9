set -x
T=r02al
timeout 600 python -m pytest tests/test_gpu_async_finish.py tests/test_gpu_graph.py tests/test_gpu_qat_step.py tests/test_gpu_host_api.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
for i in 1 2; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_async_$i.json 2>&1
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --sync-finish > gpurun_out/${T}_bench_f32_sync_$i.json 2>&1
done
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_async.json 2>&1
python tools/show_bench.py gpurun_out/${T}_bench_*.json
