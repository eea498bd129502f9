# A/B of backward kernel variants (QFB_BWD_VARIANT bits). Outputs -> gpurun_out/
timeout 300 python -m pytest tests -q -m gpu -x -k "bwd or golden" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
for v in ${VARIANTS:-0 1 2 3 4 5 6 7}; do
  for dt in ${DTYPES:-f32 f16}; do
    QFB_BWD_VARIANT=$v timeout 200 python bench.py --no-cpu --no-e2e --no-secondary --steps 300 --dtype $dt > gpurun_out/var_${v}_${dt}.json 2>/dev/null
  done
done
python tools/show_bench.py gpurun_out/var_*.json
