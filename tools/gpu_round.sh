# One gpurun call: tests, division proof, benches, ncu. Outputs -> gpurun_out/
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
if [ "${QFB_VERIFY_FULL:-0}" = "1" ]; then
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/verify_div.cu -o /tmp/verify_div && \
  timeout 900 /tmp/verify_div > gpurun_out/verify_div_full.txt 2>&1; echo rc=$? >> gpurun_out/verify_div_full.txt
fi
timeout 300 python bench.py > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
timeout 300 python bench.py --dtype f16 --no-cpu > gpurun_out/bench_f16.json 2> gpurun_out/bench_f16.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bwd|ew_|codes|perop" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
timeout 120 python tools/pcie_probe.py > gpurun_out/pcie_probe.json 2>&1
