# consumer full-barrier wait with suspend-time hints (QFB_BWD_WAIT_NS)
set -x
T=r02by
O=gpurun_out
for rep in 1 2; do
for w in 0 100 1000 10000; do
  QFB_BWD_WAIT_NS=$w timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_w${w}_$rep.json 2>&1
  QFB_BWD_WAIT_NS=$w timeout 300 python tools/bwd_only_probe.py f16 >> $O/${T}_bwd_only_w${w}.jsonl 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
cut -c1-120 $O/${T}_bwd_only_*.jsonl
