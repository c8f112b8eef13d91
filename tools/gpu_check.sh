#!/bin/bash
# One gpurun call: smoke, GPU tests, GEMM probe, bench (outputs under gpurun_out/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
if [ -n "$PROBE" ]; then timeout 900 python tools/gemm_probe.py > gpurun_out/gemm_probe.log 2>&1; fi
timeout 900 python bench.py --save-selection gpurun_out/sel_c2.json > gpurun_out/bench.log 2>&1; echo "bench rc $?" >> gpurun_out/bench.log
