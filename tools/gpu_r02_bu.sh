# packed int8 codes in the lean int8 loop: parity + A/B (QFB_FQ2)
set -x
T=r02bu
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_fwd.py tests/test_gpu_int8_out.py tests/test_gpu_frontend.py -x -q -p no:cacheprovider -k "int8 or code" > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do
for f in 1 0; do
  for dt in f32 f16; do QFB_FQ2=$f C5_REPS=40 timeout 120 python tools/c5_probe.py 8 $dt int8 >> $O/${T}_c5_fq2${f}.jsonl 2>&1; done
done
done
cut -c1-120 $O/${T}_c5_*.jsonl
