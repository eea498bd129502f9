# Fast safety-first round: smoke (short timeout) before anything long.
set -x
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
if grep -q "smoke ok" gpurun_out/smoke.log; then
  timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
  timeout 300 python bench.py > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
  timeout 300 python bench.py --dtype f16 --no-cpu > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bwd|ew_|codes|perop" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 > gpurun_out/ncu_full.log 2>&1
fi
ls -la gpurun_out
