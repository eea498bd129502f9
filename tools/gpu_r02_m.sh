set -x
T=r02m
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_gpu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ew_tma|bwd" -s 20 -c 30 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-secondary --no-graph > /dev/null 2>&1
QFB_BWD_IMPL=tile1 timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_tile1.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32.json 2>&1
tail -3 gpurun_out/${T}_pytest_gpu.log
