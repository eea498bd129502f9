set -x
timeout 600 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider > gpurun_out/r02d_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02d_pytest.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sbwd_kernel|bwd_finish" -s 2 -c 2 -o gpurun_out/r02d_sbwd python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > gpurun_out/r02d_ncu.log 2>&1
tail -3 gpurun_out/r02d_pytest.log
