# shared-memory tiled cosine kernel: parity + config-4 A/B (QFB_COSINE_TILE)
set -x
T=r02bf
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_qat_step.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for tile in 1 0; do
  QFB_COSINE_TILE=$tile timeout 300 python tools/qat_split.py > $O/${T}_split_tile$tile.json 2>&1
  QFB_COSINE_TILE=$tile timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $O/${T}_bench_tile$tile.json 2>&1
done
cat $O/${T}_split_tile*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02bf_bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); s=(d.get("secondary") or {}).get("c4_qat_step") or {}
    print(f, {k:(round(v,4) if isinstance(v,float) else v) for k,v in s.items() if k in ("ms_per_step","frames_per_s","hbm_frac")})
PY
