# config-1 per-tensor launch: TMA ring vs register-pipelined kernel, stages
set -x
T=r02bj
O=gpurun_out
for rep in 1 2; do
  timeout 120 python tools/c1_probe.py >> $O/${T}_c1_default.jsonl 2>&1
  QFB_DISABLE_TMA_FWD=1 timeout 120 python tools/c1_probe.py >> $O/${T}_c1_notma.jsonl 2>&1
  QFB_FWD_STAGES=3 timeout 120 python tools/c1_probe.py >> $O/${T}_c1_ns3.jsonl 2>&1
done
tail -n 2 $O/${T}_c1_*.jsonl
