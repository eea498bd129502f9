# f32 one-output lean loop (tools/bin/libqfb_one.so, 54 regs -> 4 CTAs/SM) vs default two-output loop
set -x
T=r02bn
O=gpurun_out
QFB_LIB_PATH=$PWD/tools/bin/libqfb_one.so timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > $O/${T}_pytest_one.log 2>&1; echo rc=$? >> $O/${T}_pytest_one.log
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest_one.log $O/${T}_pytest.log
for rep in 1 2; do
for lib in one def; do
  if [ $lib = one ]; then export QFB_LIB_PATH=$PWD/tools/bin/libqfb_one.so; else unset QFB_LIB_PATH; fi
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_${lib}_$rep.json 2>&1
  C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f32 >> $O/${T}_c5_${lib}.jsonl 2>&1
  timeout 120 python tools/c1_probe.py >> $O/${T}_c1_${lib}.jsonl 2>&1
done
done
unset QFB_LIB_PATH
python tools/show_bench.py $O/${T}_bench_*.json
cut -c1-120 $O/${T}_c5_*.jsonl $O/${T}_c1_*.jsonl
