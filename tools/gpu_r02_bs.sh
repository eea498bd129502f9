# packed f32x2 GELU polynomial in the lean chain loop: parity + config-3 A/B (QFB_FQ2)
set -x
T=r02bs
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider -k "chain or gelu or half_fast" > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for dt in f32 f16; do
for f in 1 0; do
  QFB_FQ2=$f timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --dtype $dt > $O/${T}_bench_${dt}_fq2${f}_$rep.json 2>&1
done
done
done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02bs_bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("secondary") or {}
    print(f, {k:round(v.get("gbps",0)) for k,v in s.items() if isinstance(v,dict) and "c3" in k})
PY
