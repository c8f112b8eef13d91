#!/bin/bash
# One gpurun call: whole paper models at their paper input sizes (bs 1): tune (compile on
# the box, profile, BLP), time the chosen orchestration and the operator-aligned one, and
# check the output against the fp64 oracle.  MODELS overrides the list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KORCH_MODEL_CACHE=/tmp/korch_model_cache
nproc > gpurun_out/nproc.txt
timeout ${MODELS_TIMEOUT:-3000} python bench.py --models ${MODELS:-candy,yolox,efficientvit,segformer} --no-scaled \
  --no-bw-variant --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/models.log 2>&1
echo "models rc $?" >> gpurun_out/models.log
