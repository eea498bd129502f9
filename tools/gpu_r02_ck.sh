# screened 4-stage ring: bench secondary lines (config 5 as specified, config 4) with both builds
set -x
T=r02ck
O=gpurun_out
for rep in 1 2; do
for lib in s4 def; do
  if [ $lib = s4 ]; then export QFB_LIB_PATH=$PWD/tools/bin/libqfb_s4.so; else unset QFB_LIB_PATH; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > $O/${T}_bench_${lib}_$rep.json 2>&1
done
done
unset QFB_LIB_PATH
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r02ck_bench_*.json")):
    d=json.loads(open(f).read().strip().splitlines()[-1]); s=d.get("secondary") or {}
    print(f, round(d["ms_per_step"],4), {k:round(v.get("value",v.get("gbps",v.get("ms_per_step",0))),1) for k,v in s.items() if isinstance(v,dict)}, d["clocks"]["reasons"])
PY
