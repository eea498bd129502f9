set -x
T=r02ae
timeout 600 python -m pytest tests/test_gpu_bwd_half_fp32.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
QFB_BWD_IMPL=tileqd timeout 600 python -m pytest tests/test_gpu_bwd_half_fp32.py -x -q -p no:cacheprovider >> gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
for i in 1 2; do
QFB_HALF_FP32=1 timeout 120 python tools/bwd_only_probe.py f16 >> gpurun_out/${T}_bwd_only.jsonl 2>&1
QFB_HALF_FP32=1 QFB_BWD_IMPL=tileqd timeout 120 python tools/bwd_only_probe.py f16 >> gpurun_out/${T}_bwd_only.jsonl 2>&1
done
timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 --half-fp32-terms > gpurun_out/${T}_bench_f16_h32.json 2>&1
grep -E "passed|failed|rc=" gpurun_out/${T}_pytest.log
cat gpurun_out/${T}_bwd_only.jsonl
python tools/show_bench.py gpurun_out/${T}_bench_*.json
