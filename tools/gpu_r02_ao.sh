set -x
T=r02ao
for dt in f32 f16; do
  for st in 2 3 4; do
    QFB_BWD_STAGES=$st QFB_BWD_RING_KB=110 timeout 120 python tools/bwd_only_probe.py $dt | sed "s/}$/, \"stages\": $st}/" >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
  QFB_BWD_STAGES=2 timeout 120 python tools/bwd_only_probe.py $dt | sed "s/}$/, \"stages\": \"2@76\"}/" >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
cat gpurun_out/${T}_bwd_only.jsonl
