#!/bin/bash
# One gpurun call: for each paper model, replay its bs-1 plan once to find its top kernels,
# then one ncu --set full capture of exactly those kernels (outputs under gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in ${MODELS:-candy efficientvit yolox segformer efficientvit2048}; do
  KORCH_EXEC_DIRECT=1 timeout 900 python tools/replay_model.py $m --steps 1 --top ${TOP:-4} --names gpurun_out/${m}_top.txt \
    --plan-out gpurun_out/${m}_plan.json > gpurun_out/${m}_replay.log 2>&1
  rx=$(paste -sd'|' gpurun_out/${m}_top.txt)
  KORCH_EXEC_DIRECT=1 timeout 900 ncu --set full --clock-control none -k "regex:${rx}" -c ${TOP:-4} -o gpurun_out/${m}_top -f \
    python tools/replay_model.py $m --steps 1 > gpurun_out/${m}_ncu.log 2>&1
done
