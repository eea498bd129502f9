# ncu of the distillation kernels (mse_leaf, cosine): stalls and throughput
set -x
T=r02cg
O=gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"mse_leaf|cosine" -s 2 -c 2 -o /tmp/${T} python tools/ncu_secondary.py f32 qat > $O/${T}_ncu.log 2>&1
python tools/summarize_profile.py /tmp/${T}.ncu-rep $O/${T}_ncu_summary.json --dtype f32 --note "distill kernels" > /dev/null 2>&1 || true
ncu -i /tmp/${T}.ncu-rep --page details --csv > /tmp/${T}_details.csv 2>&1; grep -E "Memory Throughput|DRAM Throughput|Achieved Occupancy|Registers Per|Issue Slots Busy|Eligible Warps|No Eligible|Theoretical Occupancy|Block Limit" /tmp/${T}_details.csv | cut -c1-220 > $O/${T}_details.txt
