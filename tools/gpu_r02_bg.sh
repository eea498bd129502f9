# backward tile order A/B (QFB_BWD_ORDER=rev: last tiles first)
set -x
T=r02bg
O=gpurun_out
QFB_BWD_ORDER=rev timeout 900 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_frontend.py tests/test_gpu_qat_step.py -x -q -p no:cacheprovider > $O/${T}_pytest_rev.log 2>&1; echo rc=$? >> $O/${T}_pytest_rev.log
tail -n 2 $O/${T}_pytest_rev.log
for rep in 1 2; do
for ord in rev fwd; do
  QFB_BWD_ORDER=$ord timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_${ord}_$rep.json 2>&1
done
done
for ord in rev fwd; do
  QFB_BWD_ORDER=$ord timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > $O/${T}_bench_f16_${ord}.json 2>&1
done
python tools/show_bench.py $O/${T}_bench_*.json
