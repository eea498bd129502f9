# Ring-size sweep of the backward kernel (QFB_BWD_RING_KB / QFB_BWD_STAGES). Outputs -> gpurun_out/
timeout 300 python -m pytest tests -q -m gpu -x -k "bwd or golden" > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
SWEEP=${SWEEP:-72:8 48:8 100:8 110:4 200:8}
for cfg in $SWEEP; do
  kb=${cfg%%:*}; ns=${cfg##*:}
  for dt in f32 f16; do
    QFB_BWD_RING_KB=$kb QFB_BWD_STAGES=$ns timeout 200 python bench.py --no-cpu --no-e2e --no-secondary --steps 300 --dtype $dt > gpurun_out/sweep_${kb}_${ns}_${dt}.json 2>/dev/null
  done
done
python tools/show_bench.py gpurun_out/sweep_*.json
