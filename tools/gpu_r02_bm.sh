# word-wise term select in the backward consumer: parity + A/B against tools/bin/libqfb_base.so
set -x
T=r02bm
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_sbwd.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for lib in sel16 base; do
  if [ $lib = base ]; then export QFB_LIB_PATH=$PWD/tools/bin/libqfb_base.so; else unset QFB_LIB_PATH; fi
  timeout 300 python tools/bwd_only_probe.py f32 >> $O/${T}_bwd_only_$lib.jsonl 2>&1
  timeout 300 python tools/bwd_only_probe.py f16 >> $O/${T}_bwd_only_$lib.jsonl 2>&1
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_${lib}_$rep.json 2>&1
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > $O/${T}_bench_f16_${lib}_$rep.json 2>&1
done
done
unset QFB_LIB_PATH
python tools/show_bench.py $O/${T}_bench_*.json
cut -c1-120 $O/${T}_bwd_only_*.jsonl
