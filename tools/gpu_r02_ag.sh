set -x
T=r02ag
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32.json 2>&1
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16.json 2>&1
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
python tools/show_bench.py gpurun_out/${T}_bench_*.json
tail -3 gpurun_out/${T}_bench_f32.json | head -2
