# full GPU suite + smoke after the lean binary16 forward
set -x
T=r02cl
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/${T}_pytest_gpu.log 2>&1; echo rc=$? >> $O/${T}_pytest_gpu.log
tail -3 $O/${T}_pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo rc=$? >> $O/${T}_smoke.log
tail -2 $O/${T}_smoke.log
