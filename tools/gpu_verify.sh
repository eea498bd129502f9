set -x
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/verify_div.cu -o /tmp/verify_div && timeout 600 /tmp/verify_div > gpurun_out/verify_div_full.txt 2>&1; echo rc=$? >> gpurun_out/verify_div_full.txt
bash tools/gpu_quick.sh
