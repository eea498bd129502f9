set -x
timeout 900 python -m pytest tests/test_gpu_sbwd.py tests/test_gpu_bwd.py tests/test_gpu_frontend.py tests/test_gpu_bench_shapes.py -x -q -p no:cacheprovider > gpurun_out/r02g_pytest.log 2>&1; echo rc=$? >> gpurun_out/r02g_pytest.log
for st in 2 3; do QFB_SB_STAGES=$st timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/r02g_bench_f32_s$st.json 2>&1; done
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/r02g_bench_f16.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sbwd_kernel|bwd_finish" -s 2 -c 2 -o gpurun_out/r02g_sbwd python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > gpurun_out/r02g_ncu.log 2>&1
for f in gpurun_out/r02g_bench_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['ms_per_step']*1e3,1), d['kernel_ms'], round(d['roofline']['frac'],3), round(d['roofline']['step_frac'],3))"; done
tail -3 gpurun_out/r02g_pytest.log
