set -x
T=${TAG:-r02h}
timeout 900 python -m pytest tests/test_gpu_sbwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
for st in ${STAGES:-2 3}; do QFB_SB_STAGES=$st timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_s$st.json 2>&1; done
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${KREG:-sbwd_kernel}" -s 1 -c 1 -o gpurun_out/${T}_sbwd python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > gpurun_out/${T}_ncu.log 2>&1
[ -n "$EXTRA" ] && eval "$EXTRA"
true
