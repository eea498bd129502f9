# round 2: streaming backward parity + timing
set -x
timeout 900 python -m pytest tests/test_gpu_sbwd.py tests/test_gpu_bwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > gpurun_out/r02c_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02c_pytest.log
tail -15 gpurun_out/r02c_pytest.log
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/r02c_bench_f32.json 2> gpurun_out/r02c_bench_f32.err
QFB_BWD_IMPL=tile timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/r02c_bench_f32_tile.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/r02c_bench_f16.json 2> gpurun_out/r02c_bench_f16.err
QFB_SB_STAGES=2 timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/r02c_bench_f32_s2.json 2>&1
for f in gpurun_out/r02c_bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3,1), d['kernel_ms'], round(d['roofline']['frac'],3), round(d['roofline']['step_frac'],3))"; done
