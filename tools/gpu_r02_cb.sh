# persistent low-occupancy cosine kernel (QFB_COSINE=persist|persist2): parity + QAT split
set -x
T=r02cb
O=gpurun_out
for v in persist persist2; do
  QFB_COSINE=$v timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_qat_step.py -x -q -p no:cacheprovider > $O/${T}_pytest_$v.log 2>&1; echo rc=$? >> $O/${T}_pytest_$v.log
  tail -n 2 $O/${T}_pytest_$v.log
done
for rep in 1 2; do
  for v in def persist persist2; do
    if [ $v = def ]; then unset QFB_COSINE; else export QFB_COSINE=$v; fi
    timeout 300 python tools/qat_split.py >> $O/${T}_split_$v.jsonl 2>&1
  done
done
unset QFB_COSINE
tail -n 2 $O/${T}_split_*.jsonl
