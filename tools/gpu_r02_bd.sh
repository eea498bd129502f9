# lean chain default mask: parity (default and all lean loops on) + bench
set -x
T=r02bd
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_exec.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -3 $O/${T}_pytest.log
QFB_FWD_LEAN=15 timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider -k "chain" > $O/${T}_pytest_lean15.log 2>&1; echo rc=$? >> $O/${T}_pytest_lean15.log
tail -3 $O/${T}_pytest_lean15.log
for dt in f32 f16; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --dtype $dt > $O/${T}_bench_${dt}.json 2>&1
done
python tools/show_bench.py $O/${T}_bench_*.json
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02bd_bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("secondary") or {}
    print(f, {k:round(v.get("gbps",0)) for k,v in s.items() if isinstance(v,dict) and "gbps" in v})
PY
