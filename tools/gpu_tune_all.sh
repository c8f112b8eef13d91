#!/bin/bash
# One gpurun call: re-record every tuning database the bench reads -- the five paper
# models at bs 1, the batch-8 local batch of the C3/C5 throughput leg (N = 1), and Candy's
# multi-output (N1) search -- under gpurun_out/tuning_db.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_db
export KORCH_CACHE_DIR=/tmp/korch_tune_cache
mkdir -p $KORCH_CACHE_DIR
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout ${TUNE_TIMEOUT:-2400} python tools/tune_models.py --out gpurun_out/tuning_db \
  ${MODELS:-candy efficientvit yolox segformer efficientvit2048} > gpurun_out/tune.log 2>&1
echo "tune rc $?" >> gpurun_out/tune.log
timeout ${TUNE_TIMEOUT:-2400} python tools/tune_models.py --out gpurun_out/tuning_db --batch ${BATCHES:-8} \
  ${SCALING_MODELS:-efficientvit yolox candy} > gpurun_out/tune_b.log 2>&1
echo "tune rc $?" >> gpurun_out/tune_b.log
timeout 900 python tools/tune_models.py --out gpurun_out/tuning_db --max-outputs 2 candy > gpurun_out/tune_mo.log 2>&1
echo "tune rc $?" >> gpurun_out/tune_mo.log
