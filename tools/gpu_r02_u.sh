# round-2 record run: every -m gpu test, smoke, benches (f32 full line, f16 with e2e, reference arm),
# launch list + ncu full of the step kernels, ncu of the secondary kernels, launch list of the
# benchmarked-shape tests, racecheck on the backward, full division proof. Outputs -> gpurun_out/
set -x
T=r02u
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_gpu.txt
lscpu | head -20 >> gpurun_out/${T}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_gpu.log
tail -2 gpurun_out/${T}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_f32.json 2> gpurun_out/${T}_bench_f32.err
timeout 600 python bench.py --dtype f16 --no-cpu > gpurun_out/${T}_bench_f16.json 2> gpurun_out/${T}_bench_f16.err
timeout 600 python bench.py --impl reference > gpurun_out/${T}_ref.json 2> gpurun_out/${T}_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bwd|ew_" -s 30 -c 30 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/${T}_prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > gpurun_out/${T}_ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o gpurun_out/${T}_prof_f16 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph --dtype f16 > gpurun_out/${T}_ncu_full_f16.log 2>&1
# secondary kernels: chain (relu, gelu), int8 emission, distill + adam (second, warm launch of each)
timeout 600 ncu --set full --clock-control none -k regex:"ew_tma_kernel" -s 1 -c 1 -o gpurun_out/${T}_c3_relu python tools/ncu_secondary.py f32 relu > gpurun_out/${T}_ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ew_tma_kernel" -s 1 -c 1 -o gpurun_out/${T}_c3_gelu python tools/ncu_secondary.py f32 gelu >> gpurun_out/${T}_ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"ew_tma_kernel" -s 1 -c 1 -o gpurun_out/${T}_c5_int8 python tools/ncu_secondary.py f32 int8 >> gpurun_out/${T}_ncu_sec.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"leaf_sums|halve|cosine|adam|nonfinite|fold" -o gpurun_out/${T}_c4_distill python tools/ncu_secondary.py f32 qat >> gpurun_out/${T}_ncu_sec.log 2>&1
# which forward ring instances the benchmarked-shape tests launch
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ew_tma|bwd_kernel" --csv --log-file gpurun_out/${T}_shapes_launches.csv python -m pytest tests/test_gpu_bench_shapes.py -q -p no:cacheprovider > gpurun_out/${T}_shapes.log 2>&1
# racecheck on the backward (consumer-side proxy fences)
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 200 python -m pytest tests/test_gpu_bwd.py -q -x -k "not full and not full_size and not graph" -p no:cacheprovider > gpurun_out/${T}_racecheck_bwd.log 2>&1; echo rc=$? >> gpurun_out/${T}_racecheck_bwd.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/verify_ddiv3 tools/verify_ddiv3.cu && timeout 1500 /tmp/verify_ddiv3 20000 > gpurun_out/${T}_verify_ddiv3.txt 2>&1; echo rc=$? >> gpurun_out/${T}_verify_ddiv3.txt
python tools/show_bench.py gpurun_out/${T}_bench_f32.json gpurun_out/${T}_bench_f16.json
