# backward tile order, second box: alone (back to back) and in the step
set -x
T=r02bk
O=gpurun_out
for rep in 1 2; do
for ord in rev fwd; do
  QFB_BWD_ORDER=$ord timeout 300 python tools/bwd_only_probe.py f32 >> $O/${T}_bwd_only_$ord.jsonl 2>&1
  QFB_BWD_ORDER=$ord timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_${ord}_$rep.json 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
cut -c1-200 $O/${T}_bwd_only_*.jsonl
