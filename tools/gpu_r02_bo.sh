# f32 2-stage one-output lean loop: parity + c1 / step check
set -x
T=r02bo
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_exec.py tests/test_gpu_graph.py tests/test_gpu_int8_out.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
  timeout 120 python tools/c1_probe.py >> $O/${T}_c1.jsonl 2>&1
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_$rep.json 2>&1
done
python tools/show_bench.py $O/${T}_bench_*.json
cut -c1-100 $O/${T}_c1.jsonl
