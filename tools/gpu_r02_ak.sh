set -x
T=r02ak
for dt in f32 f16; do
  for impl in tiled tile tiledu; do
    QFB_BWD_IMPL=$impl timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
  QFB_BWD_IMPL=tiledu QFB_BWD_VARIANT=9 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_VARIANT=8 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
cat gpurun_out/${T}_bwd_only.jsonl
