# Full evidence capture for profiles/: GPU tests, smoke, benches (f32 with CPU/e2e/secondary,
# f16), the launch list of the bench command, one ncu --set full capture of the hot kernels
# for f32 and f16. Outputs -> gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo rc=$? >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 600 python bench.py --dtype f16 --no-cpu --no-e2e > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bwd|ew_|codes|perop" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/prof_f16 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --dtype f16 > gpurun_out/ncu_full_f16.log 2>&1
ls -la gpurun_out
