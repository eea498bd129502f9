# ncu --set full of the backward kernel for the variants in $VARIANTS. Outputs -> gpurun_out/
for v in ${VARIANTS:-0}; do
  QFB_BWD_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bwd_kernel" -s 2 -c 1 -o gpurun_out/prof_v$v python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-secondary --sets 1 --dtype ${DT:-f32} > gpurun_out/ncu_v$v.log 2>&1
done
ls gpurun_out
