// Kernel generation for candidate kernels: PROFILING's "generate a kernel for the
// defined tensor algebra computation" half, re-designed for
// sm_100a.  Each candidate maps to one template (SURVEY.md §8(a')); a template
// specialises to CUDA source (all shapes/strides compile-time constants) that
// NVRTC compiles for sm_100a.  Several launch variants per candidate play the
// role of the paper's schedule tuning; the profiler keeps the fastest.
#pragma once
#include <string>
#include <vector>

#include "enumerate.h"
#include "ir.h"

namespace korch {

struct TmaDesc {            // a 2-5D TMA tensor map the host encodes per launch
  int tensor = -1;          // index into KernelPlan::ext (or -2 = output, -3 = the kernel's scratch)
  int rank = 0;
  int64_t dims[5] = {0};    // elements, innermost first
  int64_t strides[5] = {0}; // bytes, for dims 1..rank-1 (innermost stride is 1 element)
  int64_t elem_off = 0;     // element offset of the view into the tensor
  uint32_t box[5] = {0};
  int dtype = 1;            // 0 = f32, 1 = bf16
  int swizzle = 3;          // CU_TENSOR_MAP_SWIZZLE_128B
};

struct KernelVariant {
  std::string name;
  std::string source;
  int block = 256;
  int64_t grid = 1;
  int64_t grid_y = 1, grid_z = 1;
  int smem = 0;             // dynamic shared memory bytes
  int cluster = 1;
  bool tcgen05 = false;     // source needs templates/sm100_gemm.cuh ahead of it
  int64_t scratch_bytes = 0;  // library-owned, zero-initialised, self-cleaning device scratch
                              // (split-K partial sums); passed right after `out`
  std::string tag;
  std::vector<TmaDesc> tma; // passed (in order) after the pointer params
};

struct KernelPlan {
  int klass = 0;            // KORCH_CLASS_*
  std::string reject;       // reason if rejected
  std::vector<Ref> ext;     // external tensors, in kernel-parameter order
  std::vector<KernelVariant> variants;
  int64_t bytes = 0;
  double flops = 0;
};

KernelPlan generate_kernel(const Graph& g, const Candidate& c);

// Epilogue of a GEMM candidate, emitted by the row-template machinery: `body` computes
// the output chunk from float acc[32] (row gm, columns nb..nb+31) and `store` writes it.
// A full-tile side input of a GEMM epilogue (e.g. the residual of x + W.h) whose view is
// affine: element (gm, j) at off + gm * sm + j (+ batch terms).  The GEMM kernel stages
// the [128 x BN] tile by TMA into shared memory during the main loop; the epilogue reads
// it from there (`sside<i>` = its shared address, row pitch BN elements).
struct EpiSide {
  int slot = -1;                       // index into GemmEpilogue::ext
  int64_t off = 0, sm = 0;             // elements
  std::vector<int64_t> bcoef;          // per GEMM batch axis (elements)
  int dtype = 1;                       // 0 = f32, 1 = bf16
};

struct GemmEpilogue {
  std::vector<Ref> ext;               // pre_ext first, then epilogue operands
  std::string body, store;
  int64_t bytes = 0;                  // epilogue reads + output write
  std::vector<std::string> batch_vars;
  bool rows_unit = false;             // output address has unit stride along the row gm
  std::vector<EpiSide> sides;         // side inputs read from TMA-staged tiles (stage_bn > 0)
};
// t > 1: t threads share each row chunk (column-lane epilogue, see gemm_gen.cpp); the
// body then reads float acc[cw / t] for columns nb + (tid + k*t)*8 + [0, 8).
// target >= 0: compute that intermediate node instead of the candidate's output; then
// `store` holds the name of the float[cw] array with its values (no global store).
bool make_gemm_epilogue(const Graph& g, const Candidate& c, int mm, int cw, const std::vector<Ref>& pre_ext,
                        GemmEpilogue* out, std::string* err, int target = -1, int t = 1, int stage_bn = 0);
// Prologue of a GEMM whose A operand is computed in the kernel (e.g. LayerNorm feeding a
// Linear): `body` runs once per A row (local row r, global row gm; one warp per row,
// lane = tid) and writes the bf16 row into the resident, 128B-swizzled K-major A tile at
// shared address `sA`.
struct GemmPrologue {
  std::vector<Ref> ext;               // pre_ext first, then prologue operands
  std::string body;
  int64_t bytes = 0;                  // prologue reads (the A tile never reaches HBM)
  std::vector<std::string> batch_vars;
  int stage_slot = -1;                // ext slot of the tensor TMA-loaded into the A tile (-1: none)
};
bool make_gemm_prologue(const Graph& g, const Candidate& c, int mm, const std::vector<Ref>& pre_ext,
                        GemmPrologue* out, std::string* err);
KernelPlan generate_attention(const Graph& g, const Candidate& c);   // gemm_gen.cpp (N2)
KernelPlan generate_gemm(const Graph& g, const Candidate& c);   // gemm_gen.cpp
std::string kernel_prelude();
// Kernel parameters of a candidate's secondary outputs (N1, reading A32): ", T* __restrict__
// out1, ..." in the order of Candidate::extra_outputs, passed right after `out`.
std::string extra_out_params(const Graph& g, const Candidate& c);
std::string fmt_float(double v);
uint64_t fnv1a(const std::string& s);

}  // namespace korch
