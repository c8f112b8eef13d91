#!/bin/bash
# One gpurun call: tune C2 at batch 64, then ncu (launch list + --set full) on a replay.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/save_selection.py c2 64 gpurun_out/sel_c2_b64.json > gpurun_out/sel_b64.log 2>&1
export KORCH_EXEC_DIRECT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_b64.csv \
  python tools/replay.py gpurun_out/sel_c2_b64.json --steps 3 > gpurun_out/ncu_launches_b64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:korch_ -c 6 -o gpurun_out/c2_b64_full -f \
  python tools/replay.py gpurun_out/sel_c2_b64.json --steps 1 > gpurun_out/ncu_full_b64.log 2>&1
echo done >> gpurun_out/ncu_full_b64.log
