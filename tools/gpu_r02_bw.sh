# backward tail evict_last (QFB_L2_HINTS=48 = 16|32) vs default 16
set -x
T=r02bw
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_bwd.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2 3; do
for h in 16 48; do
  QFB_L2_HINTS=$h timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_h${h}_$rep.json 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
