# round-2 record run (lean outputs: every .ncu-rep is summarized on the box and only the
# headline backward/forward capture is kept). Outputs -> gpurun_out/
set -x
T=r02w
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_gpu.txt
lscpu | head -20 >> $O/${T}_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bwd_half_fp32.py tests/test_gpu_sbwd.py tests/test_gpu_dropin.py -q -p no:cacheprovider > $O/${T}_pytest_new.log 2>&1; echo rc=$? >> $O/${T}_pytest_new.log
QFB_HALF_FP32=1 timeout 120 python tools/bwd_only_probe.py f16 > $O/${T}_bwd_only_h32.jsonl 2>&1
timeout 120 python tools/bwd_only_probe.py f16 >> $O/${T}_bwd_only_h32.jsonl 2>&1
timeout 120 python tools/bwd_only_probe.py f32 >> $O/${T}_bwd_only_h32.jsonl 2>&1
timeout 900 python bench.py > $O/${T}_bench_f32.json 2> $O/${T}_bench_f32.err
timeout 600 python bench.py --dtype f16 --no-cpu > $O/${T}_bench_f16.json 2> $O/${T}_bench_f16.err
timeout 600 python bench.py --dtype f16 --no-cpu --no-secondary --half-fp32-terms > $O/${T}_bench_f16_h32.json 2> $O/${T}_bench_f16_h32.err
timeout 600 python bench.py --impl reference > $O/${T}_ref.json 2> $O/${T}_ref.err
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"bwd|ew_" -s 30 -c 30 --csv --log-file $O/${T}_launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-secondary --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o $O/${T}_prof python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph > $O/${T}_ncu_full.log 2>&1
python tools/summarize_profile.py $O/${T}_prof.ncu-rep $O/${T}_ncu_summary.json --launches $O/${T}_launches.csv --traffic profiles/ncu_traffic.json --dtype f32 --note "r02 record run, f32 step kernels" > /dev/null
cp profiles/ncu_traffic.json $O/${T}_ncu_traffic.json
timeout 600 ncu --set full --clock-control none -k regex:"bwd_kernel|ew_tma_kernel" -s 4 -c 2 -o /tmp/${T}_prof_f16 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --no-graph --dtype f16 > $O/${T}_ncu_full_f16.log 2>&1
python tools/summarize_profile.py /tmp/${T}_prof_f16.ncu-rep $O/${T}_ncu_summary_f16.json --note "r02 record run, f16 step kernels" > /dev/null
# secondary kernels (warm second launch of each; summaries only)
for w in relu gelu int8; do
  timeout 600 ncu --set full --clock-control none -k regex:"ew_tma_kernel" -s 1 -c 1 -o /tmp/${T}_$w python tools/ncu_secondary.py f32 $w >> $O/${T}_ncu_sec.log 2>&1
  python tools/summarize_profile.py /tmp/${T}_$w.ncu-rep $O/${T}_ncu_summary_$w.json --note "r02 secondary: $w" > /dev/null
done
timeout 600 ncu --set full --clock-control none -k regex:"leaf_sums|halve|cosine|adam|nonfinite" -s 8 -c 8 -o /tmp/${T}_qat python tools/ncu_secondary.py f32 qat >> $O/${T}_ncu_sec.log 2>&1
python tools/summarize_profile.py /tmp/${T}_qat.ncu-rep $O/${T}_ncu_summary_qat.json --note "r02 secondary: distill + adam (config 4)" > /dev/null
# which instances the benchmarked-shape tests launch
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ew_tma|bwd_kernel" --csv --log-file /tmp/${T}_shapes.csv python -m pytest tests/test_gpu_bench_shapes.py -q -p no:cacheprovider > $O/${T}_shapes.log 2>&1
python - <<'PY' > $O/${T}_shapes_kernels.txt
import csv, collections
rows = list(csv.reader(open("/tmp/r02w_shapes.csv")))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]; ni = h.index("Kernel Name")
c = collections.Counter(r[ni] for r in rows[i + 1:])
for k, v in sorted(c.items()): print(v, k)
PY
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 100 python -m pytest tests/test_gpu_bwd.py -q -x -k "not full and not full_size and not graph" -p no:cacheprovider > /tmp/${T}_racecheck.log 2>&1; echo rc=$? >> /tmp/${T}_racecheck.log
tail -c 20000 /tmp/${T}_racecheck.log > $O/${T}_racecheck_bwd_tail.log
grep -c "Race reported" /tmp/${T}_racecheck.log >> $O/${T}_racecheck_bwd_tail.log
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/verify_ddiv3 tools/verify_ddiv3.cu && timeout 1500 /tmp/verify_ddiv3 20000 > $O/${T}_verify_ddiv3.txt 2>&1; echo rc=$? >> $O/${T}_verify_ddiv3.txt
du -sh $O
python tools/show_bench.py $O/${T}_bench_*.json
