#!/bin/bash
# Diagnostics: one pytest case with the per-launch profile trace, then the SegFormer trace.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KORCH_PROFILE_TRACE=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${TEST_K:-c2_pipeline and kw1}" \
  > gpurun_out/trace_test.log 2> gpurun_out/trace_test_err_full.log
echo "rc $?" >> gpurun_out/trace_test.log
tail -c 6000 gpurun_out/trace_test_err_full.log > gpurun_out/trace_test_err.log; rm -f gpurun_out/trace_test_err_full.log
TRACE_TIMEOUT=900 bash tools/gpu_trace.sh
