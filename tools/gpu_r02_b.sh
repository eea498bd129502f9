# round 2: memory-pipeline probe + sanitizer runs (graph/workspace hardening, bwd proxy fence)
set -x
timeout 300 ./tools/bin/pipe_probe > gpurun_out/r02b_pipe_probe.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_graph.py -q -x -p no:cacheprovider > gpurun_out/r02b_memcheck_graph.log 2>&1; echo rc=$? >> gpurun_out/r02b_memcheck_graph.log
timeout 600 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_bwd.py -q -x -p no:cacheprovider -k "ragged_lengths and 4097" > gpurun_out/r02b_racecheck_bwd.log 2>&1; echo rc=$? >> gpurun_out/r02b_racecheck_bwd.log
tail -5 gpurun_out/r02b_memcheck_graph.log gpurun_out/r02b_racecheck_bwd.log
