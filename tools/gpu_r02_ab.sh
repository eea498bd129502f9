# fused finish: parity (every backward test), then step A/B vs the separate finisher
set -x
T=r02ab
timeout 1200 python -m pytest tests/test_gpu_sbwd.py tests/test_gpu_bwd.py tests/test_gpu_frontend.py tests/test_gpu_bench_shapes.py tests/test_gpu_qat_step.py tests/test_gpu_graph.py tests/test_gpu_golden.py tests/test_gpu_dropin.py tests/test_gpu_bwd_half_fp32.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -3 gpurun_out/${T}_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
for i in 1 2; do
  timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_fused_$i.json 2>&1
  QFB_BWD_FUSED_FIN=0 timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > gpurun_out/${T}_bench_f32_sep_$i.json 2>&1
done
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_fused.json 2>&1
for dt in f32 f16; do
  timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  QFB_BWD_FUSED_FIN=0 timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
C5_REPS=40 timeout 120 python tools/c5_probe.py 8 > gpurun_out/${T}_c5.jsonl 2>&1
C5_REPS=4000 timeout 300 python tools/c5_probe.py 8 >> gpurun_out/${T}_c5.jsonl 2>&1
cat gpurun_out/${T}_bwd_only.jsonl gpurun_out/${T}_c5.jsonl
python tools/show_bench.py gpurun_out/${T}_bench_*.json
