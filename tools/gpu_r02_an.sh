# the production structure's memory-only / arithmetic-only probes, main pass alone
set -x
T=r02an
for dt in f32 f16; do
  timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_VARIANT=2088 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_VARIANT=2096 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
cat gpurun_out/${T}_bwd_only.jsonl
