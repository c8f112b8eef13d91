#!/bin/bash
# One gpurun call for a kernel iteration: targeted GPU tests (PYTEST_K), the C2 bench line
# alone (no models / scaling / batch 64 unless BENCH_ARGS says so), and the ncu launch
# list + full capture of the C2 plan (outputs under gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$PYTEST_K" ]; then
  timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q -x -k "$PYTEST_K" > gpurun_out/pytest_iter.log 2>&1
  echo "pytest rc $?" >> gpurun_out/pytest_iter.log
fi
timeout ${BENCH_TIMEOUT:-900} python bench.py --models '' --scaling-models '' --no-bw-variant --no-cpu-baseline ${BENCH_ARGS} \
  --save-selection gpurun_out/sel_c2.json > gpurun_out/bench_iter.log 2>gpurun_out/bench_iter.err
echo "bench rc $?" >> gpurun_out/bench_iter.err
if [ -z "$SKIP_NCU" ]; then
  export KORCH_EXEC_DIRECT=1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/replay.py gpurun_out/sel_c2.json --steps 3 > gpurun_out/ncu_launches.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:korch_ -c 8 -o gpurun_out/c2_full -f \
    python tools/replay.py gpurun_out/sel_c2.json --steps 2 > gpurun_out/ncu_full.log 2>&1
fi
