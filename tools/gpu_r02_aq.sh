set -x
T=r02aq
timeout 600 python -m pytest tests/test_gpu_host_api.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for cfg in "QFB_MERGE_COPY=0" "QFB_MERGE_COPY=1" "QFB_PASS_GROUP_MB=20" "QFB_PASS_GROUP_MB=40" "QFB_PASS_GROUP_MB=80" "QFB_PASS_GROUP_MB=160"; do
  tag=$(echo $cfg | tr '=' '_')
  env $cfg timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-secondary > gpurun_out/${T}_bench_$tag.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench_$tag.json').read().strip().splitlines()[-1]); print('$cfg', round(d['e2e']['value'],1))"
done
