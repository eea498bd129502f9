# step re-check: defaults vs QFB_FQ2=0 / QFB_L2_HINTS=0 on one box, with clocks
set -x
T=r02bv
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.mem,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > $O/${T}_gpu.txt
for rep in 1 2; do
  timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_def_$rep.json 2>&1
  QFB_FQ2=0 timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_fq20_$rep.json 2>&1
  QFB_L2_HINTS=0 timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_h0_$rep.json 2>&1
  QFB_L2_HINTS=0 QFB_FQ2=0 QFB_BWD_ORDER=fwd timeout 600 python bench.py --steps 400 --warmup 10 --no-cpu --no-e2e --no-secondary > $O/${T}_bench_all0_$rep.json 2>&1
done
python tools/show_bench.py $O/${T}_bench_*.json
cat $O/${T}_gpu.txt
