# round-2 final record run (lean outputs). Outputs -> gpurun_out/
set -x
T=r02j
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_gpu.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_pytest_gpu.log 2>&1; echo rc=$? >> $O/${T}_pytest_gpu.log
tail -3 $O/${T}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
timeout 900 python bench.py > $O/${T}_bench_f32.json 2> $O/${T}_bench_f32.err
timeout 600 python bench.py --dtype f16 --no-cpu > $O/${T}_bench_f16.json 2> $O/${T}_bench_f16.err
timeout 600 python bench.py --dtype f16 --no-cpu --no-secondary --half-fp32-terms > $O/${T}_bench_f16_h32.json 2> $O/${T}_bench_f16_h32.err
timeout 600 python bench.py --impl reference > $O/${T}_bench_reference.json 2> $O/${T}_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bwd|ew_" -s 30 -c 30 --csv --log-file $O/${T}_launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o /tmp/${T}_prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > $O/${T}_ncu_full.log 2>&1
python tools/summarize_profile.py /tmp/${T}_prof.ncu-rep $O/${T}_ncu_summary.json --launches $O/${T}_launches.csv --traffic profiles/ncu_traffic.json --dtype f32 --note "r02 final, f32 step kernels" > /dev/null
cp profiles/ncu_traffic.json $O/${T}_ncu_traffic.json
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_graph.py tests/test_gpu_bwd.py tests/test_gpu_bwd_half_fp32.py -q -x -k "not full and not full_size" -p no:cacheprovider > /tmp/${T}_memcheck.log 2>&1; echo rc=$? >> /tmp/${T}_memcheck.log
tail -c 4000 /tmp/${T}_memcheck.log > $O/${T}_memcheck_tail.log
timeout 300 python tools/bwd_only_probe.py f32 > $O/${T}_bwd_only.jsonl 2>&1
timeout 300 python tools/bwd_only_probe.py f16 >> $O/${T}_bwd_only.jsonl 2>&1
du -sh $O
python tools/show_bench.py $O/${T}_bench_*.json
# round-2 lean-loop evidence: GELU chain and int8 emission kernels, f16 step kernels
for w in gelu int8; do
  timeout 300 ncu --set full --clock-control none -k regex:"ew_tma_kernel" -s 1 -c 1 -o /tmp/${T}_$w python tools/ncu_secondary.py f32 $w > $O/${T}_ncu_$w.log 2>&1
  python tools/summarize_profile.py /tmp/${T}_$w.ncu-rep $O/${T}_ncu_summary_$w.json --dtype f32 --note "r02 final, $w (lean loop)" > /dev/null 2>&1 || true
done
timeout 600 ncu --set full --clock-control none -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o /tmp/${T}_f16 python bench.py --dtype f16 --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > $O/${T}_ncu_f16.log 2>&1
python tools/summarize_profile.py /tmp/${T}_f16.ncu-rep $O/${T}_ncu_summary_f16.json --dtype f16 --note "r02 final, f16 step kernels" > /dev/null 2>&1 || true
du -sh $O
