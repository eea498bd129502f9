timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_frontend.py tests/test_gpu_golden.py tests/test_gpu_qat_step.py -q -x 2>&1 | tail -3
for r in 1 2; do
for v in new checked; do
 if [ $v = checked ]; then export QFB_LIB_PATH=$PWD/ab/libqfb_checked.so; else unset QFB_LIB_PATH; fi
 for dt in f32 f16; do
 timeout 300 python bench.py --dtype $dt --no-cpu --no-e2e --no-secondary > gpurun_out/ab_${v}_${dt}_$r.json 2>/dev/null
 done
done; done
unset QFB_LIB_PATH
python tools/show_bench.py gpurun_out/ab_*.json
