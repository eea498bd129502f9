# MSE leaf kernel: 32-bit descent + all loads in flight: parity + timing
set -x
T=r02cd
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_train.py tests/test_gpu_qat_step.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > $O/${T}_pytest.log 2>&1; echo rc=$? >> $O/${T}_pytest.log
tail -n 2 $O/${T}_pytest.log
for rep in 1 2; do timeout 300 python tools/qat_split.py >> $O/${T}_split.jsonl 2>&1; done
cat $O/${T}_split.jsonl
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"mse|cosine" --csv --log-file $O/${T}_launches.csv python tools/ncu_secondary.py f32 qat > /dev/null 2>&1
