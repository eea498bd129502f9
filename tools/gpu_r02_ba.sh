# config-3 GELU chain (f32, f16): ncu with source counters, opcode histograms
set -x
T=r02ba
O=gpurun_out
for dt in f32 f16; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ew_tma_kernel" -s 1 -c 1 -o /tmp/${T}_gelu_$dt python tools/ncu_secondary.py $dt gelu > $O/${T}_ncu_$dt.log 2>&1
python tools/ncu_ops.py /tmp/${T}_gelu_$dt.ncu-rep ew_tma_kernel 30 > $O/${T}_ops_gelu_$dt.txt 2>&1
ncu -i /tmp/${T}_gelu_$dt.ncu-rep --page source --csv -k regex:ew_tma_kernel > /tmp/${T}_src.csv 2>&1; gzip -c /tmp/${T}_src.csv > $O/${T}_src_gelu_$dt.csv.gz
python tools/summarize_profile.py /tmp/${T}_gelu_$dt.ncu-rep $O/${T}_ncu_summary_gelu_$dt.json --dtype $dt --note "gelu chain" > /dev/null 2>&1 || true
done
du -sh $O
