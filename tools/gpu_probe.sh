#!/bin/bash
# One gpurun call: the GEMM variant probe only (diagnostics).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
KORCH_SEGV_TRACE=1 timeout 900 python -X faulthandler tools/gemm_probe.py > gpurun_out/gemm_probe.log 2>&1; echo "probe rc $?" >> gpurun_out/gemm_probe.log
