# backward occupancy A/B: 3 CTAs x 72 regs (default dd) vs 2 CTAs x 96 regs with deeper rings
set -x
T=r02v
timeout 600 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider -k "default or tile" > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
for dt in f32 f16; do
  QFB_BWD_IMPL=tiled timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  for kb in 76 100 110; do
    QFB_BWD_IMPL=tile2d QFB_BWD_RING_KB=$kb timeout 120 python tools/bwd_only_probe.py $dt | sed "s/}$/, \"ring_kb\": $kb}/" >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
done
cat gpurun_out/${T}_bwd_only.jsonl
timeout 600 python -m pytest tests/test_gpu_bwd_half_fp32.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest_h32.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_h32.log
tail -3 gpurun_out/${T}_pytest_h32.log
QFB_HALF_FP32=1 timeout 120 python tools/bwd_only_probe.py f16 >> gpurun_out/${T}_bwd_only.jsonl 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 --half-fp32-terms > gpurun_out/${T}_bench_f16_h32.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16.json 2>&1
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32.json 2>&1
tail -2 gpurun_out/${T}_bwd_only.jsonl
python tools/show_bench.py gpurun_out/${T}_bench_*.json
