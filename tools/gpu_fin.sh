# A/B of the finisher (QFB_FIN_SMEM: shared-memory kernel; QFB_FIN_PDL: programmatic dependent launch)
timeout 600 python -m pytest tests/test_gpu_bwd.py tests/test_gpu_graph.py -q -x 2>&1 | tail -1
QFB_FIN_SMEM=1 timeout 600 python -m pytest tests/test_gpu_bwd.py -q -x 2>&1 | tail -1
for r in 1 2 3; do for sm in 0 1; do for pdl in 1 0; do
QFB_FIN_SMEM=$sm QFB_PDL=$pdl timeout 300 python bench.py --no-cpu --no-e2e --no-secondary > gpurun_out/fin_s${sm}_p${pdl}_$r.json 2>/dev/null
done; done; done
python tools/show_bench.py gpurun_out/fin_s*.json
