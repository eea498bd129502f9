# Forward ring-depth sweep (QFB_FWD_STAGES). Outputs -> gpurun_out/fwd_*.json
for ns in ${STAGES:-2 3 4}; do for dt in f32 f16; do
  QFB_FWD_STAGES=$ns timeout 300 python bench.py --steps 300 --no-e2e --no-cpu --dtype $dt > gpurun_out/fwd_s${ns}_${dt}.json 2>/dev/null
done; done
for f in gpurun_out/fwd_s*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); sec=d['secondary']
print('$f', 'fwd %.3f bwd %.3f' % (d['roofline']['fwd_kernel']['frac'], d['roofline']['frac']), {k: round(v['hbm_frac'],3) for k,v in sec.items()})"; done
