# A/B: current libqfb.so vs ab/libqfb_old.so (QFB_LIB_PATH), f32 bench incl. secondary lines
for r in 1 2; do for v in new old; do
 if [ $v = old ]; then export QFB_LIB_PATH=$PWD/ab/libqfb_old.so; else unset QFB_LIB_PATH; fi
 timeout 300 python bench.py --no-cpu --no-e2e > gpurun_out/ab2_${v}_$r.json 2>/dev/null
 python -c "
import json; d=json.loads(open('gpurun_out/ab2_${v}_$r.json').read().strip().splitlines()[-1]); s=d['secondary']
print('$v', 'step %.4f' % d['ms_per_step'], 'fwd %.1f' % (d['kernel_ms']['fwd']*1e3), 'c3 %.3f' % s['c3_chain_window_relu']['hbm_frac'], 'c5 %.0f' % s['c5_forward_throughput']['value'], 'int8 %.0f' % s['c5_forward_int8_codes']['value'], 'c4 %.2f' % s['c4_qat_step']['ms_per_step'])"
done; done
unset QFB_LIB_PATH
