#!/bin/bash
# One gpurun call: smoke, full GPU tests, compute-sanitizer pass, C2 bench (selection
# saved) and the ncu launch list + full capture of the C2 plan.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
if [ -z "$SKIP_TESTS" ]; then
  timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q --durations=15 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
fi
if [ -z "$SKIP_SAN" ]; then SAN_TIMEOUT=400 bash tools/gpu_sanitize.sh; fi
timeout 900 python bench.py --models '' --no-scaled --save-selection gpurun_out/sel_c2.json ${BENCH_ARGS} > gpurun_out/bench.log 2>gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
export KORCH_EXEC_DIRECT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/replay.py gpurun_out/sel_c2.json --steps 3 > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:korch_ -c 8 -o gpurun_out/c2_full -f \
  python tools/replay.py gpurun_out/sel_c2.json --steps 2 > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
