set -x
T=r02ap
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/zerocopy_probe.cu -o /tmp/zc && /tmp/zc > gpurun_out/${T}_zerocopy.txt 2>&1
timeout 120 python tools/pcie_probe.py > gpurun_out/${T}_pcie.json 2>&1
QFB_PASS_TIMING=1 timeout 300 python tools/e2e_probe.py > gpurun_out/${T}_e2e_probe.txt 2>&1
cat gpurun_out/${T}_zerocopy.txt gpurun_out/${T}_pcie.json; tail -20 gpurun_out/${T}_e2e_probe.txt
