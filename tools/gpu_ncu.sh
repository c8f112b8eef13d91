#!/bin/bash
# One gpurun call: GPU tests, bench (saves the C2 plan), then ncu on a replay of that plan:
# the launch list (gpu__time_duration) and one --set full capture of every plan kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -z "$NO_TESTS" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --durations=10 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --save-selection gpurun_out/sel_c2.json ${BENCH_ARGS} > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
export KORCH_EXEC_DIRECT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/replay.py gpurun_out/sel_c2.json --steps 3 > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:korch_ -c 8 -o gpurun_out/c2_full -f \
  python tools/replay.py gpurun_out/sel_c2.json --steps 2 > gpurun_out/ncu_full.log 2>&1
echo done >> gpurun_out/ncu_full.log
