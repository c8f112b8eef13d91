#!/bin/bash
# One gpurun call: smoke, GPU tests, whole-model tuning database, bench (outputs under
# gpurun_out/).  SKIP_TESTS=1 / SKIP_TUNE=1 / SKIP_BENCH=1 skip a leg; MODELS overrides
# the tuned model list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-2400} python -m pytest tests -m gpu -q --durations=25 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
fi
if [ -z "$SKIP_TUNE" ]; then
  mkdir -p gpurun_out/tuning_db
  KORCH_CACHE_DIR=/tmp/korch_tune_cache timeout ${TUNE_TIMEOUT:-3000} python tools/tune_models.py --out gpurun_out/tuning_db \
    ${MODELS:-candy efficientvit yolox segformer efficientvit2048} > gpurun_out/tune.log 2>&1
  echo "tune rc $?" >> gpurun_out/tune.log
  mkdir -p profiles/tuning_db && cp gpurun_out/tuning_db/*.json profiles/tuning_db/ 2>/dev/null
fi
if [ -z "$SKIP_BENCH" ]; then
  timeout ${BENCH_TIMEOUT:-1800} python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
fi
