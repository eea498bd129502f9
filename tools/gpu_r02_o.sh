set -x
T=r02o
for cfg in "QFB_BWD_CTAS=3" "QFB_BWD_CTAS=2 QFB_BWD_RING_KB=100" "QFB_BWD_CTAS=2 QFB_BWD_RING_KB=110" "QFB_BWD_CTAS=2 QFB_BWD_RING_KB=88" "QFB_BWD_CTAS=3 QFB_BWD_STAGES=2"; do
  tag=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_$tag.json 2>&1
  env $cfg timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_$tag.json 2>&1
done
