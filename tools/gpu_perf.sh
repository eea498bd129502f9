# Iteration loop: GPU parity tests + short benches (no CPU/e2e legs). Outputs -> gpurun_out/
set -x
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu --no-e2e --no-secondary > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 300 python bench.py --dtype f16 --no-cpu --no-e2e > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
if [ "${QFB_NCU:-0}" = "1" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 > gpurun_out/ncu_full.log 2>&1
fi
tail -2 gpurun_out/pytest_gpu.log
python - <<'P'
import json
for f in ("gpurun_out/bench_f32.json","gpurun_out/bench_f16.json"):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "fps %.0f step %.4f ms fwd %.1f us (%.3f) bwd %.1f us (%.3f)" % (d["value"], d["ms_per_step"], d["kernel_ms"]["fwd"]*1e3, d["roofline"]["fwd_kernel"]["frac"], d["kernel_ms"]["bwd"]*1e3, d["roofline"]["frac"]))
    except Exception as e: print(f, "ERR", e)
P
