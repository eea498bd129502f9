# same-box A/B of the config-3 chain window lines: current libqfb.so vs ab/libqfb_old.so
for r in 1 2; do for lib in new old; do
 if [ $lib = old ]; then export QFB_LIB_PATH=$PWD/ab/libqfb_old.so; else unset QFB_LIB_PATH; fi
 python bench.py --no-cpu --no-e2e > gpurun_out/c3ab_${lib}_$r.json 2>/dev/null
 python -c "
import json
d=json.loads(open('gpurun_out/c3ab_${lib}_$r.json').read().strip().splitlines()[-1]); s=d['secondary']
print('$lib', 'c3 %.3f gelu %.3f c5 %.3f int8 %.3f step %.4f' % (s['c3_chain_window_relu']['hbm_frac'], s['c3_chain_window_gelu']['hbm_frac'], s['c5_forward_throughput']['hbm_frac'], s['c5_forward_int8_codes']['hbm_frac'], d['ms_per_step']))"
done; done
unset QFB_LIB_PATH
