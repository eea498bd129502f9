# dd-quotient proof run + parity of every consumer layout + backward-alone A/B
set -x
T=r02t
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/verify_ddiv3 tools/verify_ddiv3.cu
timeout 900 python -m pytest tests/test_gpu_sbwd.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest.log
tail -2 gpurun_out/${T}_pytest.log
for dt in f32 f16; do
  for impl in tile tilem tiled tilemd tileq tileqm tileqmd; do
    QFB_BWD_IMPL=$impl timeout 120 python tools/bwd_only_probe.py $dt >> gpurun_out/${T}_bwd_only.jsonl 2>&1
  done
done
cat gpurun_out/${T}_bwd_only.jsonl
timeout 1200 /tmp/verify_ddiv3 > gpurun_out/${T}_verify_ddiv3.txt 2>&1; echo rc=$? >> gpurun_out/${T}_verify_ddiv3.txt
timeout 300 /tmp/verify_ddiv3 8 1 > gpurun_out/${T}_verify_ddiv3_control.txt 2>&1; echo rc=$? >> gpurun_out/${T}_verify_ddiv3_control.txt
cat gpurun_out/${T}_verify_ddiv3*.txt
