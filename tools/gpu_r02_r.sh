# FP64/conversion pipe throughput probe + ncu full capture of the backward (f32, f16)
set -x
T=r02r
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/fp64_probe tools/fp64_probe.cu && /tmp/fp64_probe > gpurun_out/${T}_fp64_probe.txt 2>&1
for dt in f32 f16; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel" -s 3 -c 1 -o gpurun_out/${T}_bwd_${dt} python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph --dtype $dt > gpurun_out/${T}_ncu_${dt}.log 2>&1
done
cat gpurun_out/${T}_fp64_probe.txt
