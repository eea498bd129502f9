set -x
T=r02am
for w in 1 4 8; do
  QFB_FIN_WARPS=$w timeout 600 python -m pytest tests/test_gpu_bwd.py -x -q -p no:cacheprovider -k "not full" > gpurun_out/${T}_pytest_$w.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_$w.log
  QFB_FIN_WARPS=$w timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_w$w.json 2>&1
done
tail -n 2 gpurun_out/${T}_pytest_*.log
python tools/show_bench.py gpurun_out/${T}_bench_*.json
