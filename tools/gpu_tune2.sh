#!/bin/bash
# One gpurun call: targeted GPU tests, the tuning databases (bs 1 for the five paper
# models, local batches for the C3/C5 batch sweep), then the full bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_db
nproc > gpurun_out/nproc.txt
if [ -n "$TESTS" ]; then
  timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -q --durations=10 -k "$TESTS" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
fi
export KORCH_CACHE_DIR=/tmp/korch_tune_cache
mkdir -p $KORCH_CACHE_DIR
timeout ${TUNE1_TIMEOUT:-2400} python tools/tune_models.py --out gpurun_out/tuning_db ${MODELS:-candy efficientvit yolox segformer efficientvit2048} > gpurun_out/tune.log 2>&1
echo "tune rc $?" >> gpurun_out/tune.log
if [ -n "$BATCHES" ]; then
  timeout ${TUNE2_TIMEOUT:-1500} python tools/tune_models.py --out gpurun_out/tuning_db --batch $BATCHES ${BMODELS:-efficientvit yolox candy} >> gpurun_out/tune.log 2>&1
  echo "tune batches rc $?" >> gpurun_out/tune.log
fi
unset KORCH_CACHE_DIR
mkdir -p profiles/tuning_db && cp gpurun_out/tuning_db/*.json profiles/tuning_db/
if [ -z "$SKIP_BENCH" ]; then
  timeout ${BENCH_TIMEOUT:-1500} python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
fi
