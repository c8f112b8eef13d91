#!/bin/bash
# One gpurun call after a kernel-family change: targeted GPU tests, then probes of the new
# launch variants (outputs under gpurun_out/val/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/val
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x -k "${PYTEST_K}" > gpurun_out/val/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/val/pytest.log
timeout 600 python tools/layout_probe.py > gpurun_out/val/layout_probe.log 2>&1
timeout 600 python tools/conv_probe.py candy --prefix korch_tconv --cands 5,2874,2731 > gpurun_out/val/conv_probe_candy.log 2>&1
timeout 600 python tools/conv_probe.py yolox --prefix korch_tconv --cands 27 > gpurun_out/val/conv_probe_yolox.log 2>&1
timeout 600 python tools/cand_probe.py c2 430 > gpurun_out/val/attn_probe.log 2>&1
timeout 600 python tools/cand_probe.py c2 79 664 --batch 64 > gpurun_out/val/b64_probe.log 2>&1
