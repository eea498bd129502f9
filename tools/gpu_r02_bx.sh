# f32 backward: executed count of the spill instructions (LDL/STL) from ncu source counters
set -x
T=r02bx
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel" -s 2 -c 1 -o /tmp/${T}_f32 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > $O/${T}_ncu.log 2>&1
python tools/ncu_ops.py /tmp/${T}_f32.ncu-rep bwd_kernel 40 > $O/${T}_ops_bwd_f32.txt 2>&1
ncu -i /tmp/${T}_f32.ncu-rep --page source --csv -k regex:bwd_kernel > /tmp/${T}_src.csv 2>&1; gzip -c /tmp/${T}_src.csv > $O/${T}_src_bwd_f32.csv.gz
