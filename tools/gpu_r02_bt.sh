# packed f32x2 FQ in every lean fast path: parity + A/B (QFB_FQ2)
set -x
T=r02bt
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_frontend.py tests/test_gpu_exec.py tests/test_gpu_graph.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for f in 1 0; do
  QFB_FQ2=$f timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_f32_fq2${f}_$rep.json 2>&1
  QFB_FQ2=$f timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --dtype f16 > $O/${T}_sec_f16_fq2${f}_$rep.json 2>&1
  QFB_FQ2=$f C5_REPS=40 timeout 120 python tools/c5_probe.py 8 f32 >> $O/${T}_c5_fq2${f}.jsonl 2>&1
  QFB_FQ2=$f timeout 120 python tools/c1_probe.py >> $O/${T}_c1_fq2${f}.jsonl 2>&1
done
done
python tools/show_bench.py $O/${T}_bench_*.json
