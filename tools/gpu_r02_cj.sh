# 4-stage ring with the screened packed fast path (tools/bin/libqfb_s4.so) vs default: config 5 sustained + burst
set -x
T=r02cj
O=gpurun_out
QFB_LIB_PATH=$PWD/tools/bin/libqfb_s4.so timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_bench_shapes.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for lib in s4 def; do
  if [ $lib = s4 ]; then export QFB_LIB_PATH=$PWD/tools/bin/libqfb_s4.so; else unset QFB_LIB_PATH; fi
  C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f32 >> $O/${T}_c5_$lib.jsonl 2>&1
  C5_REPS=4000 timeout 300 python tools/c5_probe.py 8 f32 >> $O/${T}_c5long_$lib.jsonl 2>&1
done
done
unset QFB_LIB_PATH
cut -c1-120 $O/${T}_c5*.jsonl
