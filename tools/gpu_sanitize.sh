# compute-sanitizer over the device parity tests at their reduced sizes
# (full-size cases deselected: the tools slow kernels 10-100x).
# memcheck: out-of-bounds / misaligned global+shared accesses, leaks at exit;
# synccheck: illegal barrier use; racecheck: shared-memory hazards (the
# mbarrier/TMA handoffs are invisible to it, so its reports on the TMA
# kernels are read by hand). Outputs -> gpurun_out/sanitize_*.log
set -x
SEL='not full and not full_size and not graph'
T="tests/test_gpu_fwd.py tests/test_gpu_bwd.py tests/test_gpu_int8_out.py tests/test_gpu_train.py tests/test_gpu_exec.py tests/test_gpu_host_api.py"
timeout 1500 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 --target-processes all \
  python -m pytest $T -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_memcheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_memcheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 \
  python -m pytest tests/test_gpu_fwd.py tests/test_gpu_bwd.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_synccheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_synccheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard \
  python -m pytest tests/test_gpu_bwd.py tests/test_gpu_fwd.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/sanitize_racecheck.log 2>&1; echo rc=$? >> gpurun_out/sanitize_racecheck.log
tail -3 gpurun_out/sanitize_*.log
