set -x
T=r02ar
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ew_tma_kernel" -s 3 -c 1 -o gpurun_out/${T}_fwd16 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph --dtype f16 > gpurun_out/${T}_ncu.log 2>&1
