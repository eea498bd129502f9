# A/B of programmatic dependent launch per edge (QFB_PDL bit mask: 1 fwd, 2 bwd, 4 finisher)
for m in 0 4 1 2 5 6; do
QFB_PDL=$m timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/pdlm${m}_f32.json 2>/dev/null
python -c "
import json,sys; d=json.loads(open('gpurun_out/pdlm${m}_f32.json').read().strip().splitlines()[-1]); s=d['secondary']
print('mask $m', 'step %.4f ms' % d['ms_per_step'], 'fwd %.1f bwd %.1f' % (d['kernel_ms']['fwd']*1e3, d['kernel_ms']['bwd']*1e3), 'c1 %.2f us' % s['c1_per_tensor_fwd']['us_per_call_rotating'], 'c4 %.2f ms' % s['c4_qat_step']['ms_per_step'], 'c5 %.0f' % s['c5_forward_throughput']['value'])"
done
