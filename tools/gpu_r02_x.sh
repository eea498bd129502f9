# ncu of the f16 float32-term backward (quad layout) and the quad memory-only probe
set -x
T=r02x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel" -s 3 -c 1 -o gpurun_out/${T}_h32 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph --dtype f16 --half-fp32-terms > gpurun_out/${T}_ncu.log 2>&1
ls -la gpurun_out
