# warp-specialized forward ring: parity + A/B against the previous build (tools/bin/libqfb_base.so)
set -x
T=r02bi
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_int8_out.py tests/test_gpu_bench_shapes.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for lib in ws base; do
  if [ $lib = base ]; then export QFB_LIB_PATH=$PWD/tools/bin/libqfb_base.so; else unset QFB_LIB_PATH; fi
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_${lib}_$rep.json 2>&1
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > $O/${T}_bench_f16_${lib}_$rep.json 2>&1
  C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f32 >> $O/${T}_c5_${lib}.jsonl 2>&1
  C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f16 >> $O/${T}_c5_${lib}.jsonl 2>&1
done
done
unset QFB_LIB_PATH
python tools/show_bench.py $O/${T}_bench_*.json
cut -c1-160 $O/${T}_c5_*.jsonl
