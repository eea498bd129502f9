set -x
T=r02av
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider -k "f16 or half or 1" > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for lean in 1 0; do
  QFB_FWD_LEAN=$lean timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > gpurun_out/${T}_bench_f16_lean$lean.json 2>&1
  QFB_FWD_LEAN=$lean C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f16 >> gpurun_out/${T}_c5.jsonl 2>&1
done
python tools/show_bench.py gpurun_out/${T}_bench_*.json; cut -c1-150 gpurun_out/${T}_c5.jsonl
