# summarize a round-2 probe: tests, bench lines, ncu metrics of the sbwd kernel
T=$1
tail -2 gpurun_out/${T}_pytest.log | head -1
for f in gpurun_out/${T}_bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3,1), {k:round(v*1e3,1) for k,v in d['kernel_ms'].items()}, round(d['roofline']['frac'],3), round(d['roofline']['step_frac'],3))"; done
ncu -i gpurun_out/${T}_sbwd.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin))
hdr=rows[0]
for r in rows[2:]:
  d={h:r[i] for i,h in enumerate(hdr)}
  print(d['Kernel Name'][:40], 'us', d['gpu__time_duration.sum'], 'inst', d.get('smsp__inst_executed.sum'), 'fp64%', d['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'], 'issue%', d['smsp__issue_active.avg.pct_of_peak_sustained_active'], 'warps%', d['sm__warps_active.avg.pct_of_peak_sustained_active'], 'dram%', d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'], 'regs', d['launch__registers_per_thread'], 'grid', d['launch__grid_size'])
st=[(float(rows[2][i]),h.replace('smsp__average_warps_issue_stalled_','').replace('_per_issue_active.ratio','')) for i,h in enumerate(hdr) if 'smsp__average_warps_issue_stalled' in h and 'per_issue_active' in h and rows[2][i]]
print(sorted(st,reverse=True)[:7])
"
