#!/bin/bash
# One gpurun call: batch tuning databases for the C3/C5 sweep (local batches), the N = 1
# bench line, and a 2-rank run on the one GPU with the gloo backend (exercises the
# multi-rank paths G1-G4 and the rank spawning of bench.py --gpus 2).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_db
if [ -n "$BATCHES" ]; then
  KORCH_CACHE_DIR=/tmp/korch_tune_cache timeout ${TUNE2_TIMEOUT:-1500} python tools/tune_models.py --out gpurun_out/tuning_db --batch $BATCHES ${BMODELS:-efficientvit yolox candy} > gpurun_out/tune_b.log 2>&1
  echo "tune batches rc $?" >> gpurun_out/tune_b.log
  mkdir -p profiles/tuning_db && cp gpurun_out/tuning_db/*.json profiles/tuning_db/
fi
timeout ${BENCH_TIMEOUT:-1200} python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
if [ -z "$SKIP_N2" ]; then
  KORCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline ${N2_ARGS} > gpurun_out/bench_n2.log 2>gpurun_out/bench_n2.err; echo "bench n2 rc $?" >> gpurun_out/bench_n2.err
fi
