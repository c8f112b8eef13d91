#!/bin/bash
# One gpurun call: compute-sanitizer memcheck / racecheck / synccheck on one small instance
# of each kernel template family (row PW/RR, column CR, staged transpose TR, tcgen05 GEMM
# incl. cluster split-K, persistent GEMM, implicit-GEMM conv, fused attention, multi-output
# epilogues), through the same pytest parity cases (outputs under gpurun_out/sanitize_*).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SEL='test_c1_shapes_whole_and_singletons and 37-100 or test_transpose_tiles_every_variant and 2-45-70 and bf16 or test_column_reductions_every_variant and ReduceSum-f32 or test_every_gemm_variant and 128-768-768 or test_persistent_gemm_every_variant and 256-64-1024 or test_conv_igemm_every_variant and shape0 or test_fused_attention_candidates and kw0 or test_gemm_epilogue_secondary_outputs and bf16'
for tool in memcheck racecheck synccheck; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --error-exitcode 17 --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi_output.py -q -x -k "$SEL" \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc $?" >> gpurun_out/sanitize_$tool.log
done
