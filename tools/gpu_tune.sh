#!/bin/bash
# One gpurun call: tune the paper's whole models on the B200 and record the tuning
# database (tools/tune_models.py) under gpurun_out/tuning_db (copied to
# profiles/tuning_db afterwards).  MODELS overrides the list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_db
export KORCH_CACHE_DIR=/tmp/korch_tune_cache
mkdir -p $KORCH_CACHE_DIR
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout ${TUNE_TIMEOUT:-3000} python tools/tune_models.py --out gpurun_out/tuning_db \
  ${MODELS:-candy efficientvit yolox segformer efficientvit2048} > gpurun_out/tune.log 2>&1
echo "tune rc $?" >> gpurun_out/tune.log
