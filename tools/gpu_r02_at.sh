set -x
T=r02at
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_bench_shapes.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for lean in 1 0 1; do
  QFB_FWD_LEAN=$lean timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_lean$lean.json 2>&1
  python tools/show_bench.py gpurun_out/${T}_bench_f32_lean$lean.json
done
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16.json 2>&1
python tools/show_bench.py gpurun_out/${T}_bench_f16.json
