timeout 300 python -m pytest tests/test_gpu_bwd.py -q -x 2>&1 | tail -2
for v in 8 16; do for dt in f32 f16; do
QFB_BWD_VARIANT=$v timeout 300 python bench.py --dtype $dt --no-cpu --no-e2e --no-secondary > gpurun_out/probe_${v}_${dt}.json 2>/dev/null
done; done
python tools/show_bench.py gpurun_out/probe_*.json
