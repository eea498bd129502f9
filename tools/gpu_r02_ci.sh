# TMA chunk size A/B (QFB_FWD_CHUNK units: 1024 default, 512, 256)
set -x
T=r02ci
O=gpurun_out
QFB_FWD_CHUNK=512 timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > $O/${T}_pytest512.log 2>&1; echo rc=$? >> $O/${T}_pytest512.log
tail -n 2 $O/${T}_pytest512.log
for rep in 1 2; do
for c in 1024 512 256; do
  QFB_FWD_CHUNK=$c timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_c${c}_$rep.json 2>&1
  QFB_FWD_CHUNK=$c timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > $O/${T}_bench_f16_c${c}_$rep.json 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
