# consumer wait suspend hints under sustained (power-capped) runs: 1000 and 4000 steps
set -x
T=r02cm
O=gpurun_out
for rep in 1 2; do
for w in 0 1000; do
  QFB_BWD_WAIT_NS=$w timeout 600 python bench.py --steps 4000 --warmup 50 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_w${w}_4k_$rep.json 2>&1
  QFB_BWD_WAIT_NS=$w timeout 600 python bench.py --steps 1000 --warmup 20 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_w${w}_1k_$rep.json 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
