# f16 step kernels: ncu full capture with source counters, opcode histograms
set -x
T=r02ay
O=gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o /tmp/${T}_f16 python bench.py --dtype f16 --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > $O/${T}_ncu.log 2>&1
python tools/ncu_ops.py /tmp/${T}_f16.ncu-rep ew_tma_kernel 40 > $O/${T}_ops_fwd_f16.txt 2>&1
ncu -i /tmp/${T}_f16.ncu-rep --page source --csv -k regex:ew_tma_kernel > /tmp/${T}_src_fwd.csv 2>&1; gzip -c /tmp/${T}_src_fwd.csv > $O/${T}_src_fwd_f16.csv.gz
du -sh $O
python tools/summarize_profile.py /tmp/${T}_f16.ncu-rep $O/${T}_ncu_summary_f16.json --dtype f16 --note "lean f16 forward" > /dev/null 2>&1 || true
