# CTA-uniform backward (bwd_cu_kernel): parity, then memory-only and full vs the warp-specialized kernel
set -x
T=r02ai
timeout 900 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider -k "tiledu" > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for dt in f32 f16; do
  QFB_BWD_IMPL=tiled timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_IMPL=tiledu timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_IMPL=tiledu QFB_BWD_VARIANT=9 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  for st in 2 4; do
    QFB_BWD_IMPL=tiledu QFB_BWD_STAGES=$st QFB_BWD_RING_KB=100 timeout 120 python tools/bwd_only_probe.py $dt | sed "s/}$/, \"stages\": $st}/" >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
done
cat gpurun_out/${T}_bwd_only.jsonl
