# drop-in harness on the GPU + streaming vs tile backward, f32/f16
set -x
T=r02q
timeout 600 python -m pytest tests/test_gpu_dropin.py -x -q -p no:cacheprovider > gpurun_out/${T}_dropin.log 2>&1; echo rc=$? >> gpurun_out/${T}_dropin.log
./oracle/_ref/dropin_frontend >> gpurun_out/${T}_dropin.log 2>&1
for impl in tile stream; do
  for dt in f32 f16; do
    QFB_BWD_IMPL=$impl timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype $dt > gpurun_out/${T}_bench_${dt}_${impl}.json 2>&1
  done
done
for f in gpurun_out/${T}_bench_*.json; do python tools/show_bench.py $f; done
