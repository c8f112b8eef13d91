#!/bin/bash
# One gpurun call: the default bench line (N = 1), a 2-rank gloo run on the one GPU, the
# ncu launch list + full capture of the C2 plan, and ncu captures of every paper model's
# top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout ${BENCH_TIMEOUT:-1500} python bench.py --save-selection gpurun_out/sel_c2.json > gpurun_out/bench.log 2>gpurun_out/bench.err
echo "bench rc $?" >> gpurun_out/bench.err
if [ -z "$SKIP_N2" ]; then
  KORCH_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-bw-variant \
    --models candy,efficientvit --scaling-models candy \
    > gpurun_out/bench_n2.log 2>gpurun_out/bench_n2.err; echo "bench n2 rc $?" >> gpurun_out/bench_n2.err
fi
export KORCH_EXEC_DIRECT=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python tools/replay.py gpurun_out/sel_c2.json --steps 3 > gpurun_out/ncu_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:korch_ -c 8 -o gpurun_out/c2_full -f \
  python tools/replay.py gpurun_out/sel_c2.json --steps 2 > gpurun_out/ncu_full.log 2>&1
unset KORCH_EXEC_DIRECT
TOP=${TOP:-3} bash tools/gpu_ncu_models.sh
