set -x
T=r02aj
for dt in f32 f16; do
  for v in 9 10 11; do
    QFB_BWD_IMPL=tiledu QFB_BWD_VARIANT=$v timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
done
QFB_BWD_IMPL=tiledu QFB_BWD_VARIANT=11 timeout 600 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider -k "tiledu" > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
cat gpurun_out/${T}_bwd_only.jsonl; tail -2 gpurun_out/${T}_pytest.log
