#!/bin/bash
# One gpurun call: a list of tuning jobs "model:batch[:mo]" (env JOBS), each recorded into
# gpurun_out/tuning_db and copied into profiles/tuning_db; optional bench afterwards.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/tuning_db profiles/tuning_db
export KORCH_CACHE_DIR=/tmp/korch_tune_cache
mkdir -p $KORCH_CACHE_DIR
for job in $JOBS; do
  IFS=: read -r m b mo <<< "$job"
  timeout ${JOB_TIMEOUT:-900} python tools/tune_models.py --out gpurun_out/tuning_db --batch $b --max-outputs ${mo:-1} $m >> gpurun_out/tune.log 2>&1
  echo "job $job rc $?" >> gpurun_out/tune.log
  cp gpurun_out/tuning_db/*.json profiles/tuning_db/ 2>/dev/null
done
unset KORCH_CACHE_DIR
if [ -n "$BENCH" ]; then
  timeout ${BENCH_TIMEOUT:-1200} python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
fi
if [ -n "$N2" ]; then
  KORCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline ${N2_ARGS} > gpurun_out/bench_n2.log 2>gpurun_out/bench_n2.err; echo "bench n2 rc $?" >> gpurun_out/bench_n2.err
fi
