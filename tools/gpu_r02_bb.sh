# lean chain loop: parity + config-3 A/B (QFB_FWD_LEAN)
set -x
T=r02bb
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -3 $O/${T}_pytest.log
for dt in f32 f16; do
for lean in 1 0; do
  QFB_FWD_LEAN=$lean timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --dtype $dt > $O/${T}_bench_${dt}_lean${lean}.json 2>&1
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02bb_bench_*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("secondary") or {}
        print(f, {k:(round(v.get("frac",0),3), round(v.get("value",0),1)) for k,v in s.items() if isinstance(v,dict) and "c3" in k})
    except Exception as e: print(f, e)
PY
