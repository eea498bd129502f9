# lean binary16 forward (one output at a time): parity + A/B (QFB_FWD_LEAN)
set -x
T=r02ax
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_int8_out.py tests/test_gpu_exec.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -2 $O/${T}_pytest.log
for rep in 1 2; do
for lean in 1 0; do
  QFB_FWD_LEAN=$lean timeout 300 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary --dtype f16 > $O/${T}_bench_f16_lean${lean}_$rep.json 2>&1
done
done
for lean in 1 0; do
  QFB_FWD_LEAN=$lean C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f16 >> $O/${T}_c5.jsonl 2>&1
done
python tools/show_bench.py $O/${T}_bench_*.json; cut -c1-200 $O/${T}_c5.jsonl
