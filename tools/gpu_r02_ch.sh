# f16 backward: magic-number rint (QFB_BWD_IMPL=tilemd) with the word-wise select, vs default
set -x
T=r02ch
O=gpurun_out
for rep in 1 2; do
for impl in default tilemd; do
  if [ $impl = default ]; then unset QFB_BWD_IMPL; else export QFB_BWD_IMPL=$impl; fi
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > $O/${T}_bench_f16_${impl}_$rep.json 2>&1
done
done
unset QFB_BWD_IMPL
python tools/show_bench.py $O/${T}_bench_*.json
