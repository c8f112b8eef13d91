#!/bin/bash
# Full GPU suite with a per-launch profile trace kept (tail) in case of a hang.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KORCH_PROFILE_TRACE=1 KORCH_SEGV_TRACE=1 timeout ${T:-1500} python -m pytest tests -m gpu -q -s -p no:cacheprovider \
  > gpurun_out/pytest_gpu.log 2> gpurun_out/pytest_err_full.log
echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
tail -c 8000 gpurun_out/pytest_err_full.log > gpurun_out/pytest_err_tail.log; rm -f gpurun_out/pytest_err_full.log
