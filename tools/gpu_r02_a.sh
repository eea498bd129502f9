# round 2, first GPU pass: every -m gpu test, then the default bench (N=1) and the reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r02a_pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02a_ref.json 2> gpurun_out/r02a_ref.err
tail -3 gpurun_out/r02a_pytest_gpu.log
