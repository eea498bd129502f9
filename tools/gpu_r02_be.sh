# lean int8 emission: parity + A/B (QFB_FWD_LEAN 29 = default, 13 = int8 general)
set -x
T=r02be
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_int8_out.py tests/test_gpu_bench_shapes.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for dt in f32 f16; do
for lean in 29 13; do
  QFB_FWD_LEAN=$lean timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu --no-e2e --dtype $dt > $O/${T}_bench_${dt}_lean${lean}_$rep.json 2>&1
done
done
done
python tools/show_bench.py $O/${T}_bench_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02be_bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("secondary") or {}
    print(f, {k:round(v.get("value",0)) for k,v in s.items() if isinstance(v,dict) and "c5" in k})
PY
