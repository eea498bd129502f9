set -x
timeout 300 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_bwd.py -q -x -k "ragged_lengths and (4097 or 76800) or per_channel_axis0 or multi_table" > gpurun_out/sanitize_memcheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_memcheck.log
timeout 300 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_bwd.py -q -x -k "ragged_lengths and 4097" > gpurun_out/sanitize_racecheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_racecheck.log
timeout 300 compute-sanitizer --tool synccheck python -m pytest tests/test_gpu_bwd.py -q -x -k "ragged_lengths and 4097" > gpurun_out/sanitize_synccheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_synccheck.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bwd|ew_|codes|perop" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 > gpurun_out/ncu_full.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench_f32.json 2> gpurun_out/bench_f32.err
QFB_DISABLE_TMA_FWD=1 timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/bench_f32_notma.json 2>&1
ls -la gpurun_out
