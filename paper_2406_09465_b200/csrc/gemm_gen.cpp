// KB5: GEMM template for candidates with exactly one dense linear primitive (MatMul /
// batched MatMul), the paper's "compute-intensive" class, re-designed for
// sm_100a: tcgen05.mma (bf16 in, fp32 accumulate in TMEM), operands staged by TMA into a
// multi-stage mbarrier ring with 128B swizzle, one 128 x BN tile per CTA (or a persistent
// tile loop, see the persistent variant).
//
// Upstream members (Transpose / Reshape / Slice chains feeding the MatMul) are folded
// into the TMA tensor maps as strided views -- the data-layout trick of P:529-531
// (kernel k5) without materialising the transposed operand.  Downstream members
// (elementwise ops, port broadcasts, side-branch reads, Transpose/Reshape of the result)
// are fused into the epilogue, emitted by the row-template machinery.
#include <algorithm>
#include <set>
#include <sstream>

#include "../../include/korch.h"
#include "codegen.h"
#include "expr.h"

namespace korch {

extern const char* kSm100GemmTemplate;  // templates/sm100_gemm.cuh (embedded by build.py)

namespace {

struct View {
  Ref src;                      // external tensor
  std::vector<int64_t> coef;    // per operand axis (batch..., row, col), elements
  int64_t off = 0;              // element offset
  Shape shape;                  // operand shape
  // K-split view: the contraction axis k addresses (k % ksplit) * coef[k axis] +
  // (k / ksplit) * kout, e.g. the head-merge Transpose+Reshape in front of an attention
  // output projection (A[s, h*64 + d] = O[h, s, d]).  A 64-wide K-block never straddles
  // a split when ksplit % 64 == 0, so TMA loads it as one box of a rank+1 tensor map.
  int64_t ksplit = 0, kout = 0;
};

bool operand_view(const Graph& g, const std::set<int>& mem, const Prim& L, int slot, View* v, std::set<int>* chain,
                  std::string* err) {
  ExprCtx X;
  const Shape& s = g.shape_of(L.in[slot]);
  std::vector<Lin> co;
  std::vector<int> vars;
  for (size_t i = 0; i < s.size(); ++i) {
    int id = X.add_var("a" + std::to_string(i), 0, s[i] - 1);
    vars.push_back(id);
    co.push_back(X.var(id));
  }
  Ref r = L.in[slot];
  while (!r.is_input && mem.count(r.id)) {
    const Prim& q = g.prims[r.id];
    chain->insert(q.id);
    const Shape& is = g.shape_of(q.in[0]);
    std::vector<Lin> c2;
    if (q.kind == Kind::Transpose) {
      c2.resize(co.size());
      for (size_t i = 0; i < co.size(); ++i) c2[q.perm[i]] = co[i];
    } else if (q.kind == Kind::Reshape) {
      Lin flat = ExprCtx::cst(0);
      int64_t st = 1;
      for (int k = (int)q.shape.size() - 1; k >= 0; --k) {
        flat = ExprCtx::add(flat, ExprCtx::scale(co[k], st));
        st *= q.shape[k];
      }
      c2.resize(is.size());
      st = 1;
      for (int k = (int)is.size() - 1; k >= 0; --k) {
        c2[k] = X.mod(X.div(flat, st), is[k]);
        st *= is[k];
      }
    } else if (q.kind == Kind::Slice) {
      c2 = co;
      c2[q.axis] = ExprCtx::add(co[q.axis], ExprCtx::cst(q.start));
    } else {
      *err = std::string("'") + kind_name(q.kind) + "' upstream of the linear primitive is not a strided view";
      return false;
    }
    co = c2;
    r = q.in[0];
  }
  const Shape& ts = g.shape_of(r);
  Lin addr = ExprCtx::cst(0);
  int64_t st = 1;
  for (int k = (int)ts.size() - 1; k >= 0; --k) {
    addr = ExprCtx::add(addr, ExprCtx::scale(co[k], st));
    st *= ts[k];
  }
  // the contraction axis: A = [.., M, K] (last), B = [.., K, N] (second to last)
  const int kax = slot == 0 ? (int)s.size() - 1 : (int)s.size() - 2;
  int64_t D = 0, cdiv = 0, cmod = 0;
  for (auto& t : addr.terms) {
    const Atom& at = t.second;
    if (at.type == Atom::Var) continue;
    const bool on_k = (at.type == Atom::Div || at.type == Atom::Mod) && at.sub && at.sub->c0 == 0 &&
                      at.sub->terms.size() == 1 && at.sub->terms[0].first == 1 &&
                      at.sub->terms[0].second.type == Atom::Var && at.sub->terms[0].second.var == vars[kax];
    if (!on_k || (D && at.c != D) || s[kax] % at.c) {
      *err = "operand view is not affine (layout chain does not fold into strides)";
      return false;
    }
    D = at.c;
    (at.type == Atom::Div ? cdiv : cmod) += t.first;
  }
  v->src = r;
  v->shape = s;
  v->off = addr.c0;
  v->coef.assign(s.size(), 0);
  for (size_t i = 0; i < s.size(); ++i) {
    int64_t c = 0;
    for (auto& t : addr.terms)
      if (t.second.type == Atom::Var && t.second.var == vars[i]) c += t.first;
    v->coef[i] = c;
  }
  if (D) {  // k = D * (k / D) + k % D
    v->ksplit = D;
    v->kout = cdiv + v->coef[kax] * D;
    v->coef[kax] += cmod;
  }
  return true;
}

std::string str(int64_t v) { return std::to_string(v); }

}  // namespace

// KB6: implicit-GEMM convolution on tcgen05.  D[f, p] = sum_k W[f, k] * X_col[k, p] with
// f = output channel, p = output pixel (n, oh, ow) linearised, k = (c, r, s) in the weight's
// natural [F, C, R, S] order.  A (weights) streams by TMA (K-major, 128B swizzle); the
// im2col operand B is gathered by four producer warps straight from the NCHW input into
// the canonical MN-major 128B-swizzled shared-memory layout (zero padding, strides and the
// K tail as predicated loads), published to the tensor core with fence.proxy.async and an
// mbarrier; one thread issues the MMAs; the fused epilogue is the GEMM template's.
// The B operand of a gather GEMM: element (k, p) of the [K, NP] operand is read from
// external tensor `src` by the code in `elem` (defines `ok` and `idx` from kg, p).
struct GatherSpec {
  Ref a_src, b_src;
  int64_t M = 0, NP = 0, K = 0;
  int64_t a_off = 0, a_row = 0;   // A = [M, K] K-major view: element offset, row stride (elements)
  std::string elem;               // per-element gather code
  std::string prologue;           // per-k code shared by the 8 elements of a group
  // optional vector path: code defining `vok` (the group's 8 elements are 8 consecutive
  // in-bounds bf16 of the source) and `vidx` (index of the first); the group is then read
  // with two aligned 16-byte loads and a funnel shift instead of 8 scalar loads
  std::string vec;
  std::string tag;
  std::string prefix;             // kernel name prefix
  int64_t b_bytes = 0;            // algorithmic bytes of B
};


// Fused epilogue over a 128 x BN TMEM accumulator tile.  Warp w (< 4) owns TMEM lanes
// 32w..32w+31 = tile rows tile_m + 32w + lane; `ep` was emitted with
// make_gemm_epilogue(cw = CW, t = T).
//  * T == 1 (row mapping): each thread runs the epilogue on its own row, CW columns per
//    pass; coalesced when the output is contiguous along rows (ep.rows_unit).
//  * T > 1 (column-lane mapping): each CW-column chunk goes TMEM -> registers -> the warp's
//    slice of a shared staging buffer (pitch CW + 4 floats, conflict-free 16-byte writes
//    and reads) and is re-read with T lanes per row, so one warp instruction of the side
//    reads and of the store covers 32/T rows of 8T contiguous columns instead of 32 rows
//    of 16 bytes.  The staging buffer aliases the operand ring, which is idle once the
//    accumulator barrier has fired (every TMA load was consumed by an MMA before it).
// tcgen05.alloc takes a power of two >= 32 columns (BN = 160 for an in-tile row
// reduction over N = 160 allocates 256)
static int tmem_cols(int n) {
  int c = 32;
  while (c < n) c <<= 1;
  return c;
}
static int stage_pitch(int CW) { return CW + 4; }
static int stage_bytes(int CW) { return 4 * 32 * stage_pitch(CW) * 4; }

static std::string emit_tmem_epilogue(const GemmEpilogue& ep, int BN, int CW, int T, int64_t M, int64_t N,
                                      const std::string& tmem = "tmem", const std::string& wq = "warp",
                                      const std::string& stg_base = "smem") {
  std::ostringstream k;
  auto tmem_load = [&](const char* dst) {
    std::ostringstream t;
    if (CW <= 32) {
      t << "      tc_ld" << CW << "(" << tmem << " + ((unsigned)(" << wq << " * 32) << 16) + (unsigned)(ch * " << CW << "), " << dst
        << ");\n";
    } else {
      t << "      #pragma unroll\n      for (int q = 0; q < " << CW / 32 << "; ++q)\n"
        << "        tc_ld32(" << tmem << " + ((unsigned)(" << wq << " * 32) << 16) + (unsigned)(ch * " << CW << " + q * 32), " << dst
        << " + q * 32);\n";
    }
    return t.str();
  };
  if (T == 1) {
    k << "  {\n    const int gm = tile_m + " << wq << " * 32 + lane;\n    const int tid = 0;\n    (void)tid;\n";
    k << "    #pragma unroll 1\n    for (int ch = 0; ch < " << BN / CW << "; ++ch) {\n";
    k << "      const int nb = tile_n + ch * " << CW << ";\n";
    k << "      float acc[" << CW << "];\n";
    k << tmem_load("acc");
    k << "      if (gm < " << M << " && nb < " << N << ") {\n";
    k << ep.body << ep.store;
    k << "      }\n    }\n  }\n";
    return k.str();
  }
  const int P = stage_pitch(CW), R = 32 / T;
  k << "  {\n    float* stg = reinterpret_cast<float*>(" << stg_base << ") + " << wq << " * " << 32 * P << ";\n";
  k << "    const int tid = lane % " << T << ", rsub = lane / " << T << ";\n";
  k << "    #pragma unroll 1\n    for (int ch = 0; ch < " << BN / CW << "; ++ch) {\n";
  k << "      const int nb = tile_n + ch * " << CW << ";\n";
  k << "      if (nb >= " << N << ") break;  // chunk wholly past N (uniform)\n";
  k << "      {\n        float accr[" << CW << "];\n";
  k << tmem_load("accr");
  k << "        #pragma unroll\n        for (int q = 0; q < " << CW / 4 << "; ++q)\n";
  k << "          *reinterpret_cast<float4*>(stg + lane * " << P << " + 4 * q) = "
       "make_float4(accr[4 * q], accr[4 * q + 1], accr[4 * q + 2], accr[4 * q + 3]);\n      }\n";
  k << "      __syncwarp();\n";
  // Rows past M (ragged last tile) compute on a clamped row and skip the store, so every
  // pass's side reads are unconditional and the unrolled passes keep their loads in
  // flight together (columns past N: whole chunks are skipped above, a partial chunk is
  // masked inside the body, N % CW != 0).
  k << "      #pragma unroll\n      for (int pp = 0; pp < " << T << "; ++pp) {\n";
  k << "        const int rl = pp * " << R << " + rsub;\n";
  k << "        const int gmr = tile_m + " << wq << " * 32 + rl;\n";
  k << "        const int gm = gmr < " << M << " ? gmr : " << M - 1 << ";\n";
  k << "        float acc[8];\n";
  k << "        {\n          const float4 a0 = *reinterpret_cast<const float4*>(stg + rl * " << P << " + tid * 8);\n";
  k << "          const float4 a1 = *reinterpret_cast<const float4*>(stg + rl * " << P << " + tid * 8 + 4);\n";
  k << "          acc[0] = a0.x; acc[1] = a0.y; acc[2] = a0.z; acc[3] = a0.w;\n";
  k << "          acc[4] = a1.x; acc[5] = a1.y; acc[6] = a1.z; acc[7] = a1.w;\n        }\n";
  k << "        {\n" << ep.body << "        if (gmr < " << M << ") {\n" << ep.store << "        }\n        }\n";
  k << "      }\n      __syncwarp();\n    }\n  }\n";
  return k.str();
}


// Cluster split-K reduction (KS CTAs of a cluster hold K-slice partials of one 128 x BN
// tile in TMEM).  (1) cluster barrier: every CTA's MMAs are done, so every operand ring
// is idle and becomes a receive buffer [KS slots][RO rows][BN (+4 pad)] fp32 at `smem`;
// (2) each epilogue thread (warp quarter `wq`, lane = row within it) pushes its
// accumulator row into the owner CTA of that row (rows [o*RO, (o+1)*RO) belong to rank
// o) with st.shared::cluster; (3) cluster barrier (release/acquire); (4) the owner sums
// the KS slots of its RO rows and runs the fused epilogue `ep` (emitted with cw = BN,
// t = BN/8) with T = BN/8 lanes per row.  `epi_cond` selects the threads that own TMEM
// rows (the epilogue warps); every thread of the CTA must execute this code (the cluster
// barriers are .aligned over all threads).  No global scratch, no atomics.
static std::string emit_dsmem_splitk(const GemmEpilogue& ep, int BN, int CW, int KS, int64_t M, int64_t N,
                                     const std::string& epi_cond, const std::string& wq, int nthreads) {
  std::ostringstream k;
  const int RO = 128 / KS, PB = BN + 4, TE = BN / 8;
  k << "  cluster_sync();\n";
  k << "  if (" << epi_cond << ") {\n    const int r = " << wq << " * 32 + lane;\n";
  k << "    const unsigned dst = cluster_map(smem_u32(smem) + (unsigned)((ks * " << RO << " + r % " << RO << ") * "
    << PB * 4 << "), (unsigned)(r / " << RO << "));\n";
  k << "    #pragma unroll 1\n    for (int ch = 0; ch < " << BN / CW << "; ++ch) {\n";
  k << "      float accr[" << CW << "];\n";
  k << "      tc_ld" << CW << "(tmem + ((unsigned)(" << wq << " * 32) << 16) + (unsigned)(ch * " << CW << "), accr);\n";
  k << "      #pragma unroll\n      for (int q = 0; q < " << CW / 4 << "; ++q)\n";
  k << "        st_cluster_v4(dst + (unsigned)((ch * " << CW << " + 4 * q) * 4), accr[4 * q], accr[4 * q + 1], "
       "accr[4 * q + 2], accr[4 * q + 3]);\n";
  k << "    }\n  }\n";
  k << "  cluster_sync();\n";
  k << "  {\n    const float* recv = reinterpret_cast<const float*>(smem);\n";
  k << "    #pragma unroll\n    for (int it = threadIdx.x; it < " << RO * TE << "; it += " << nthreads << ") {\n";
  k << "      const int rl = it / " << TE << ", tid = it % " << TE << ";\n";
  k << "      const int gmr = tile_m + ks * " << RO << " + rl;\n";
  k << "      const int gm = gmr < " << M << " ? gmr : " << M - 1 << ";\n";
  k << "      const int nb = tile_n;\n";
  k << "      float acc[8];\n";
  k << "      #pragma unroll\n      for (int e = 0; e < 8; ++e) acc[e] = 0.f;\n";
  k << "      #pragma unroll\n      for (int sl = 0; sl < " << KS << "; ++sl) {\n";
  k << "        const float* src = recv + (sl * " << RO << " + rl) * " << PB << " + tid * 8;\n";
  k << "        const float4 a0 = *reinterpret_cast<const float4*>(src), a1 = *reinterpret_cast<const float4*>(src + 4);\n";
  k << "        acc[0] += a0.x; acc[1] += a0.y; acc[2] += a0.z; acc[3] += a0.w;\n";
  k << "        acc[4] += a1.x; acc[5] += a1.y; acc[6] += a1.z; acc[7] += a1.w;\n      }\n";
  k << "      {\n" << ep.body << "      if (gmr < " << M << ") {\n" << ep.store << "      }\n      }\n";
  k << "    }\n  }\n";
  return k.str();
}

// The same reduction without cluster barriers on the critical path: the receive buffer
// `recv` ([KS][RO][BN + 4] fp32) is a region of its own (not the operand ring), and
// `rbar` (count 1, armed with the (KS - 1) * RO * BN * 4 remote bytes and published to the
// cluster by a barrier before the programmatic-dependency wait) completes when every
// peer's partial rows have landed: peers push with st.async ... mbarrier::complete_tx
// into the owner's slot, the owner's own slot is written locally and published by a
// 128-thread named barrier.  Every CTA is the owner of RO rows, so none exits before the
// pushes into its shared memory completed.
static std::string emit_dsmem_splitk_async(const GemmEpilogue& ep, int BN, int CW, int KS, int64_t M, int64_t N,
                                           const std::string& recv, const std::string& rbar) {
  std::ostringstream k;
  const int RO = 128 / KS, PB = BN + 4, TE = BN / 8;
  k << "  if (warp < 4) {\n  {\n    const int r = warp * 32 + lane, owner = r / " << RO << ";\n";
  k << "    const unsigned loc = smem_u32(" << recv << ") + (unsigned)((ks * " << RO << " + r % " << RO << ") * " << PB * 4
    << ");\n";
  k << "    const unsigned dst = cluster_map(loc, (unsigned)owner), dbar = cluster_map(smem_u32(" << rbar
    << "), (unsigned)owner);\n";
  k << "    #pragma unroll 1\n    for (int ch = 0; ch < " << BN / CW << "; ++ch) {\n";
  k << "      float accr[" << CW << "];\n";
  k << "      tc_ld" << CW << "(tmem + ((unsigned)(warp * 32) << 16) + (unsigned)(ch * " << CW << "), accr);\n";
  k << "      if (owner == ks) {\n";
  k << "        #pragma unroll\n        for (int q = 0; q < " << CW / 4 << "; ++q)\n";
  k << "          *reinterpret_cast<float4*>(" << recv << " + (ks * " << RO << " + r % " << RO << ") * " << PB * 4
    << " + (ch * " << CW << " + 4 * q) * 4) = make_float4(accr[4 * q], accr[4 * q + 1], accr[4 * q + 2], accr[4 * q + 3]);\n";
  k << "      } else {\n";
  k << "        #pragma unroll\n        for (int q = 0; q < " << CW / 4 << "; ++q)\n";
  k << "          asm volatile(\"st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];\"\n"
       "                       ::\"r\"(dst + (unsigned)((ch * " << CW << " + 4 * q) * 4)), \"f\"(accr[4 * q]), \"f\"(accr[4 * q + 1]),\n"
       "                       \"f\"(accr[4 * q + 2]), \"f\"(accr[4 * q + 3]), \"r\"(dbar) : \"memory\");\n";
  k << "      }\n    }\n  }\n";
  k << "  named_bar_sync(1, 128);\n  mbar_wait(" << rbar << ", 0);\n";
  k << "  {\n    const float* rcv = reinterpret_cast<const float*>(" << recv << ");\n";
  k << "    #pragma unroll\n    for (int it = threadIdx.x; it < " << RO * TE << "; it += 128) {\n";
  k << "      const int rl = it / " << TE << ", tid = it % " << TE << ";\n";
  k << "      const int gmr = tile_m + ks * " << RO << " + rl;\n";
  k << "      const int gm = gmr < " << M << " ? gmr : " << M - 1 << ";\n";
  k << "      const int nb = tile_n;\n";
  k << "      float acc[8];\n";
  k << "      #pragma unroll\n      for (int e = 0; e < 8; ++e) acc[e] = 0.f;\n";
  k << "      #pragma unroll\n      for (int sl = 0; sl < " << KS << "; ++sl) {\n";
  k << "        const float* src = rcv + (sl * " << RO << " + rl) * " << PB << " + tid * 8;\n";
  k << "        const float4 a0 = *reinterpret_cast<const float4*>(src), a1 = *reinterpret_cast<const float4*>(src + 4);\n";
  k << "        acc[0] += a0.x; acc[1] += a0.y; acc[2] += a0.z; acc[3] += a0.w;\n";
  k << "        acc[4] += a1.x; acc[5] += a1.y; acc[6] += a1.z; acc[7] += a1.w;\n      }\n";
  k << "      {\n" << ep.body << "      if (gmr < " << M << ") {\n" << ep.store << "      }\n      }\n";
  k << "    }\n  }\n  }\n";
  return k.str();
}

// Column-lane epilogue choice: T = CW / 8 lanes per row unless the output is contiguous
// along rows (then the row mapping already stores coalesced) or the epilogue reduces rows.
static int epilogue_lanes(const Graph& g, const Candidate& c, int mm, int CW, const std::vector<Ref>& pre,
                          int64_t ring_bytes, GemmEpilogue* ep, int stage_bn = 0) {
  if (ep->rows_unit || CW % 8 || CW > 32 || stage_bytes(CW) > ring_bytes) return 1;
  for (int m : c.members)
    if (g.prims[m].kind == Kind::Reduce) return 1;
  GemmEpilogue e2;
  std::string err;
  if (!make_gemm_epilogue(g, c, mm, CW, pre, &e2, &err, -1, CW / 8, stage_bn)) return 1;
  if (e2.ext.size() != ep->ext.size()) return 1;
  *ep = e2;
  return CW / 8;
}

static KernelPlan generate_gather_gemm(const Graph& g, const Candidate& c, int mm, const GatherSpec& gs);

static KernelPlan generate_conv_gemm(const Graph& g, const Candidate& c, int mm) {
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  const Prim& L = g.prims[mm];
  std::set<int> mem(c.members.begin(), c.members.end());
  for (int m : c.members)
    for (int p : g.preds[m])
      if (m == mm && mem.count(p)) {
        kp.reject = "conv operand computed inside the candidate";
        return kp;
      }
  const Ref& xr = L.in[0];
  const Ref& wr = L.in[1];
  if (!xr.is_input && mem.count(xr.id)) { kp.reject = "conv input computed inside the candidate"; return kp; }
  if (g.dtype_of(xr) != DType::BF16 || g.dtype_of(wr) != DType::BF16) {
    kp.reject = "conv operands must be bf16";
    return kp;
  }
  if (L.groups != 1) { kp.reject = "grouped convolution"; return kp; }
  const Shape& xs = g.shape_of(xr);
  const Shape& ws = g.shape_of(wr);
  const Shape& ys = L.shape;
  int64_t Cin = xs[1], H = xs[2], W = xs[3], F = ws[0], R = ws[2], S = ws[3];
  int64_t K = Cin * R * S, OH = ys[2], OW = ys[3], NP = ys[0] * OH * OW;
  if (K % 8) { kp.reject = "conv K = C*R*S not a multiple of 8 (TMA row stride)"; return kp; }
  GatherSpec gs;
  gs.a_src = wr;
  gs.b_src = xr;
  gs.M = F;
  gs.NP = NP;
  gs.K = K;
  gs.a_off = 0;
  gs.a_row = K;
  std::ostringstream pr, el;
  pr << "        const int ci = kg / " << R * S << ", rs = kg % " << R * S << ";\n";
  pr << "        const int rr = rs / " << S << ", ss = rs % " << S << ";\n";
  el << "          const int img = p / " << OH * OW << ", q = p % " << OH * OW << ";\n";
  el << "          const int ih = (q / " << OW << ") * " << L.stride[0] << " + rr - " << L.cpad[0] << ";\n";
  el << "          const int iw = (q % " << OW << ") * " << L.stride[1] << " + ss - " << L.cpad[1] << ";\n";
  el << "          const bool ok = kg < " << K << " && p < " << NP << " && (unsigned)ih < " << H << "u && (unsigned)iw < "
     << W << "u;\n";
  el << "          const size_t idx = (((size_t)img * " << Cin << " + ci) * " << H << " + ih) * " << W << " + iw;\n";
  gs.prologue = pr.str();
  gs.elem = el.str();
  if (L.stride[1] == 1 && OW % 8 == 0) {
    // stride-1 rows: 8 consecutive output pixels (never straddling a row since OW % 8 == 0
    // and groups start at multiples of 8) read 8 consecutive input elements of one row
    std::ostringstream ve;
    ve << "        const int p0 = tile_n + grp * 8;\n";
    ve << "        const int img0 = p0 / " << OH * OW << ", q0 = p0 % " << OH * OW << ";\n";
    ve << "        const int ih0 = (q0 / " << OW << ") * " << L.stride[0] << " + rr - " << L.cpad[0] << ";\n";
    ve << "        const int iw0 = (q0 % " << OW << ") + ss - " << L.cpad[1] << ";\n";
    ve << "        const bool vok = kg < " << K << " && p0 + 7 < " << NP << " && (unsigned)ih0 < " << H
       << "u && iw0 >= 0 && iw0 + 7 < " << W << ";\n";
    ve << "        const size_t vidx = (((size_t)img0 * " << Cin << " + ci) * " << H << " + ih0) * " << W << " + iw0;\n";
    gs.vec = ve.str();
  }
  std::ostringstream t;
  t << "conv-igemm F=" << F << " P=" << NP << " K=" << K << " (" << R << "x" << S << " s" << L.stride[0] << ")";
  gs.tag = t.str();
  gs.prefix = "korch_conv_";
  gs.b_bytes = 2 * numel(xs);
  return generate_gather_gemm(g, c, mm, gs);
}

// KB5 fallback for a 2-D MatMul whose B view has no 16-byte-aligned stride (e.g. a
// pointwise conv over H*W = 196 tokens): A by TMA, B gathered by the conv template's
// producer warps.
static KernelPlan generate_matmul_gather(const Graph& g, const Candidate& c, int mm, const View& va, const View& vb) {
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  const Prim& L = g.prims[mm];
  const Shape& C = L.shape;
  for (size_t i = 0; i + 2 < C.size(); ++i)
    if (C[i] != 1) { kp.reject = "gather GEMM: batched"; return kp; }
  const int nbA = (int)va.shape.size() - 2, nbB = (int)vb.shape.size() - 2;
  const int64_t M = C[C.size() - 2], N = C.back(), K = va.shape.back();
  if (va.ksplit || vb.ksplit) { kp.reject = "gather GEMM: K-split view"; return kp; }
  if (va.coef[nbA + 1] != 1 || (va.off * 2) % 16 || (va.coef[nbA] * 2) % 16 || va.coef[nbA] <= 0 || K % 8) {
    kp.reject = "gather GEMM: A not a 16-byte aligned K-major view";
    return kp;
  }
  GatherSpec gs;
  gs.a_src = va.src;
  gs.b_src = vb.src;
  gs.M = M;
  gs.NP = N;
  gs.K = K;
  gs.a_off = va.off;
  gs.a_row = va.coef[nbA];
  std::ostringstream el;
  el << "          const bool ok = kg < " << K << " && p < " << N << ";\n";
  el << "          const size_t idx = " << vb.off << " + (size_t)kg * " << vb.coef[nbB] << " + (size_t)p * " << vb.coef[nbB + 1]
     << ";\n";
  gs.elem = el.str();
  if (vb.coef[nbB + 1] == 1) {
    // N-contiguous B (a weight whose row pitch is not 16-byte aligned, e.g. SegFormer's
    // 150-class classifier, or a [C, HW] activation with HW = 196 / 676): a group of 8
    // consecutive columns of one K row is one unaligned 16-byte read
    std::ostringstream ve;
    ve << "        const int p0 = tile_n + grp * 8;\n";
    ve << "        const bool vok = kg < " << K << " && p0 + 7 < " << N << ";\n";
    ve << "        const size_t vidx = " << vb.off << " + (size_t)kg * " << vb.coef[nbB] << " + (size_t)p0;\n";
    gs.vec = ve.str();
  }
  std::ostringstream t;
  t << "gemm-gatherB M=" << M << " N=" << N << " K=" << K;
  gs.tag = t.str();
  gs.prefix = "korch_gg_";
  gs.b_bytes = 2 * numel(vb.shape);
  return generate_gather_gemm(g, c, mm, gs);
}

static KernelPlan generate_gather_gemm(const Graph& g, const Candidate& c, int mm, const GatherSpec& gs) {
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  for (int m : c.members)
    if (g.prims[m].kind == Kind::Reduce) { kp.reject = "gather GEMM: no in-tile row reductions"; return kp; }
  const int64_t F = gs.M, NP = gs.NP, K = gs.K;
  std::vector<Ref> pre{gs.a_src, gs.b_src};
  GemmEpilogue ep0;
  std::string err;
  if (!make_gemm_epilogue(g, c, mm, 32, pre, &ep0, &err)) {
    kp.reject = err;
    return kp;
  }
  kp.ext = ep0.ext;
  const int slotW = 0, slotX = (gs.a_src.is_input == gs.b_src.is_input && gs.a_src.id == gs.b_src.id) ? 0 : 1;
  kp.flops = 2.0 * (double)F * (double)NP * (double)K;
  kp.bytes = ep0.bytes + 2 * F * K + gs.b_bytes;
  const int64_t NK = (K + 63) / 64, Mt = (F + 127) / 128;
  // launch configurations: BN in {64, 128} unsplit; cluster split-K (KS CTAs of a cluster
  // take K-slices of NKc blocks each, the last one shorter) when the grid is small -- the
  // gathered operand dominates these kernels, and splitting K splits the gather
  // occupancy variant: a 2-stage ring (~50 KB of shared memory) lets several CTAs share an
  // SM, so more gather warps hide the scattered-load latency
  struct GCfg { int bn, ks, stages = 0; };
  std::vector<GCfg> cfgs{{64, 1}, {128, 1}, {64, 1, 2}};
  for (int ks : {2, 4, 8}) {
    const int64_t tiles = Mt * ((NP + 63) / 64), nkc = (NK + ks - 1) / ks;
    if (tiles < 148 && tiles * ks <= 2 * 148 && (ks - 1) * nkc < NK) cfgs.push_back({64, ks});
  }
  for (const GCfg& cf : cfgs) {
    const int BN = cf.bn, KS = cf.ks;
    const int64_t NKc = (NK + KS - 1) / KS;  // K-blocks per slice (the last may be shorter)
    GemmEpilogue ep;
    if (!make_gemm_epilogue(g, c, mm, KS > 1 ? BN : 32, pre, &ep, &err, -1, KS > 1 ? BN / 8 : 1)) continue;
    if (ep.ext.size() != kp.ext.size()) continue;
    const int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2, STAGE = A_BYTES + B_BYTES;
    const int S_ = cf.stages ? cf.stages : (int)std::max<int64_t>(2, std::min<int64_t>({NKc, 4, (200 * 1024) / STAGE}));
    if (cf.stages && NKc <= cf.stages) continue;  // identical to the default ring
    const int64_t recv = KS > 1 ? (int64_t)128 * (BN + 4) * 4 : 0;
    // split-K receive buffer of its own (barrier-free reduction) when shared memory allows
    const bool rasync = KS > 1 && (int64_t)S_ * STAGE + recv + 1024 + (2 * S_ + 2) * 8 + 16 <= 227 * 1024;
    const int64_t REG = rasync ? (int64_t)S_ * STAGE + recv : std::max<int64_t>((int64_t)S_ * STAGE, recv);
    const int smem = (int)REG + 1024 + (2 * S_ + 2) * 8 + 16;
    const int TE = KS > 1 ? BN / 8 : epilogue_lanes(g, c, mm, 32, pre, (int64_t)S_ * STAGE, &ep);
    const int64_t Nt = (NP + BN - 1) / BN;
    const int tcols = tmem_cols(BN);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    TmaDesc da;
    da.tensor = slotW;
    da.dtype = 1;
    da.swizzle = 3;
    da.elem_off = gs.a_off;
    da.rank = 2;
    da.dims[0] = K; da.strides[0] = 2; da.box[0] = 64;
    da.dims[1] = F; da.strides[1] = gs.a_row * 2; da.box[1] = 128;
    std::ostringstream k;
    k << "extern \"C\" __global__ void __launch_bounds__(192, 1) KNAME(";
    for (size_t i = 0; i < kp.ext.size(); ++i)
      k << "const " << (g.dtype_of(kp.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
    k << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c) << ", "
      << "const __grid_constant__ TmaMap tmA) {\n";
    k << "  typedef int idx_t;\n";
    k << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
    k << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
    k << "  unsigned long long* full = (unsigned long long*)(smem + " << REG << ");\n";
    k << "  unsigned long long* empty = full + " << S_ << ";\n";
    k << "  unsigned long long* accf = empty + " << S_ << ";\n";
    if (rasync) k << "  unsigned long long* rbar = accf + 1;\n  unsigned* tslot = (unsigned*)(accf + 2);\n";
    else k << "  unsigned* tslot = (unsigned*)(accf + 1);\n";
    k << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
    if (KS > 1)
      k << "  const int ks = blockIdx.x % " << KS << ";\n  const int tile_m = (blockIdx.x / " << KS
        << ") * 128, tile_n = blockIdx.y * " << BN << ";\n";
    else
      k << "  const int ks = 0;\n  const int tile_m = blockIdx.x * 128, tile_n = blockIdx.y * " << BN << ";\n";
    k << "  const int kb0 = ks * " << NKc << ", kb1 = kb0 + " << NKc << " < " << NK << " ? kb0 + " << NKc << " : " << NK
      << ";\n";
    k << "  if (threadIdx.x == 0) {\n    for (int s = 0; s < " << S_
      << "; ++s) { mbar_init(full + s, 5); mbar_init(empty + s, 1); }\n"
      << "    mbar_init(accf, 1);\n" << (rasync ? "    mbar_init(rbar, 1);\n" : "")
      << "    mbar_fence_init();\n    tma_prefetch(&tmA);\n";
    if (rasync) k << "    mbar_expect_tx(rbar, " << (int64_t)(KS - 1) * (128 / KS) * BN * 4 << "u);\n";
    // weights (a graph input): first PRE stages fetched before the programmatic-dependency wait
    const bool early = gs.a_src.is_input;
    if (early) {
      k << "    for (int s = 0; s < " << S_ << " && kb0 + s < kb1; ++s) {\n";
      k << "      mbar_expect_tx(full + s, " << A_BYTES << "u);\n";
      k << "      tma_load_2d(smem + s * " << STAGE << ", &tmA, full + s, (kb0 + s) * 64, tile_m);\n    }\n";
    }
    k << "  }\n";
    k << "  if (warp == 5) tc_alloc(tslot, " << tcols << ");\n";
    k << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
    k << "  const unsigned tmem = *tslot;\n";
    if (rasync) k << "  asm volatile(\"barrier.cluster.arrive.relaxed.aligned;\\nbarrier.cluster.wait.aligned;\" ::: \"memory\");\n";
    k << "  pdl_trigger();\n  pdl_wait();\n";
    // gather producers: warps 0-3
    k << "  if (warp < 4) {\n";
    k << "    const bf16_t* __restrict__ xin = p" << slotX << ";\n";
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = kb0; kb < kb1; ++kb) {\n";
    k << "      mbar_wait(empty + s, ph ^ 1u);\n";
    k << "      const unsigned sb = smem_u32(smem + s * " << STAGE << " + " << A_BYTES << ");\n";
    // two phases: every group's global loads are issued before any shared-memory store
    // (the stores are asm volatile with a memory clobber, which would otherwise serialise
    // one L2 round trip per group)
    const int ITERS = (64 * (BN / 8) + 127) / 128;
    k << "      uint4 pks[" << ITERS << "];\n";
    k << "      #pragma unroll\n      for (int itg = 0; itg < " << ITERS << "; ++itg) {\n";
    k << "        const int u = threadIdx.x + itg * 128;\n";
    k << "        const int kk = u / " << BN / 8 << ", grp = u % " << BN / 8 << ";\n";
    k << "        const int kg = kb * 64 + kk;\n";
    k << gs.prologue;
    k << "        uint4 pk = make_uint4(0u, 0u, 0u, 0u);\n";
    k << "        if (u < " << 64 * (BN / 8) << ") {\n";
    if (!gs.vec.empty()) {
      k << gs.vec;
      k << "        if (vok) {\n          pk = ld_bf16x8_unaligned(xin + vidx);\n        } else {\n";
    } else {
      k << "        {\n";
    }
    k << "        unsigned short v[8];\n";
    k << "        #pragma unroll\n        for (int e = 0; e < 8; ++e) {\n";
    k << "          const int p = tile_n + grp * 8 + e;\n";
    k << gs.elem;
    k << "          v[e] = ok ? __ldg(xin + idx) : (unsigned short)0;\n";
    k << "        }\n";
    k << "        pk.x = v[0] | ((unsigned)v[1] << 16); pk.y = v[2] | ((unsigned)v[3] << 16);\n";
    k << "        pk.z = v[4] | ((unsigned)v[5] << 16); pk.w = v[6] | ((unsigned)v[7] << 16);\n";
    k << "        }\n";
    k << "        }\n        pks[itg] = pk;\n      }\n";
    // MN-major SW128 canonical: 64-pixel atoms 8 KB apart, K rows 128 B, 16B chunk ^ (row % 8)
    k << "      #pragma unroll\n      for (int itg = 0; itg < " << ITERS << "; ++itg) {\n";
    k << "        const int u = threadIdx.x + itg * 128;\n";
    k << "        const int kk = u / " << BN / 8 << ", grp = u % " << BN / 8 << ";\n";
    k << "        if (u < " << 64 * (BN / 8) << ") st_shared_v4(sb + (grp >> 3) * 8192 + kk * 128 + (((grp & 7) ^ (kk & 7)) << 4), pks[itg]);\n";
    k << "      }\n";
    k << "      fence_async_smem();\n      __syncwarp();\n";
    k << "      if (lane == 0) mbar_arrive(full + s);\n";
    k << "      if (++s == " << S_ << ") { s = 0; ph ^= 1u; }\n    }\n";
    // weight TMA: warp 4
    k << "  } else if (warp == 4 && lane == 0) {\n";
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = kb0; kb < kb1; ++kb) {\n";
    k << "      mbar_wait(empty + s, ph ^ 1u);\n";
    k << "      if (" << (early ? "kb - kb0 >= " + str(S_) : std::string("true")) << ") {\n";
    k << "      mbar_expect_tx(full + s, " << A_BYTES << "u);\n";
    k << "      tma_load_2d(smem + s * " << STAGE << ", &tmA, full + s, kb * 64, tile_m);\n      }\n";
    k << "      if (++s == " << S_ << ") { s = 0; ph ^= 1u; }\n    }\n";
    // MMA: warp 5
    k << "  } else if (warp == 5 && lane == 0) {\n";
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = kb0; kb < kb1; ++kb) {\n";
    k << "      mbar_wait(full + s, ph);\n      tc_fence_after();\n";
    k << "      const unsigned sa = smem_u32(smem + s * " << STAGE << "), sb = sa + " << A_BYTES << ";\n";
    k << "      #pragma unroll\n      for (int k = 0; k < 4; ++k) {\n";
    k << "        const unsigned long long ad = umma_desc(sa + k * 32, 16, 1024);\n";
    k << "        const unsigned long long bd = umma_desc(sb + k * 2048, 8192, 1024);\n";
    k << "        tc_mma(tmem, ad, bd, " << idesc << "u, kb != kb0 || k != 0);\n      }\n";
    k << "      tc_commit(empty + s);\n";
    k << "      if (++s == " << S_ << ") { s = 0; ph ^= 1u; }\n    }\n";
    k << "    tc_commit(accf);\n  }\n";
    // epilogue: warps 0-3 (TMEM lane quarters 0-3)
    k << "  __syncwarp();\n";
    if (KS == 1) {
      k << "  if (warp < 4) {\n    mbar_wait(accf, 0);\n    __syncwarp();\n    tc_fence_after();\n";
      k << emit_tmem_epilogue(ep, BN, 32, TE, F, NP);
      k << "  }\n";
    } else {
      k << "  if (warp < 4) {\n    mbar_wait(accf, 0);\n    __syncwarp();\n    tc_fence_after();\n  }\n";
      if (rasync) k << emit_dsmem_splitk_async(ep, BN, 32, KS, F, NP, "(smem + " + str((int64_t)S_ * STAGE) + ")", "rbar");
      else k << emit_dsmem_splitk(ep, BN, 32, KS, F, NP, "warp < 4", "warp", 192);
    }
    k << "  tc_fence_before();\n  __syncthreads();\n";
    k << "  if (warp == 5) tc_dealloc(tmem, " << tcols << ");\n}\n";

    KernelVariant kv;
    std::string src = k.str();
    char nm[64];
    std::snprintf(nm, sizeof nm, "%s%016llx", gs.prefix.c_str(),
                  (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + src));
    kv.name = nm;
    size_t pos = src.find("KNAME");
    src.replace(pos, 5, kv.name);
    kv.source = src;
    kv.tcgen05 = true;
    kv.block = 192;
    kv.grid = Mt * KS;
    kv.grid_y = Nt;
    kv.grid_z = 1;
    kv.cluster = KS;
    kv.smem = smem;
    kv.tma = {da};
    std::ostringstream t;
    t << gs.tag << " BM=128 BN=" << BN << " BK=64 splitK=" << KS << " stages=" << S_ << (TE > 1 ? " epi=cl" : "")
      << (rasync ? " red=st.async" : "");
    kv.tag = t.str();
    kp.variants.push_back(kv);
  }
  if (!kp.variants.empty()) {
    kp.klass = KORCH_CLASS_GEMM;
    kp.reject.clear();
  }
  return kp;
}

// KB5-P: GEMM with a computed A operand (a LayerNorm / elementwise chain over K feeding
// the Linear, P:433-435's "memory-intensive + compute-intensive" fusion that library GEMMs
// cannot do).  The CTA's whole A row block [128 x K] stays resident in shared memory:
// warps 0-3 compute it row by row with the row-template emitter (one warp per row,
// shuffle reductions over K, 16-byte loads) and store bf16 straight into the canonical
// K-major 128B-swizzled layout; warp 4 streams B by TMA through a stage ring; warp 5
// issues tcgen05.mma once A is published (fence.proxy.async + mbarrier); warps 0-3 then
// run the fused epilogue from TMEM.  K <= 768 (A tile <= 192 KB).
static KernelPlan generate_prologue_gemm(const Graph& g, const Candidate& c, int mm) {
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  const Prim& L = g.prims[mm];
  std::set<int> mem(c.members.begin(), c.members.end());
  View vb;
  std::set<int> chainB;
  std::string err;
  if (L.kind != Kind::MatMul) { kp.reject = "prologue GEMM: MatMul only"; return kp; }
  if (!operand_view(g, mem, L, 1, &vb, &chainB, &err)) { kp.reject = "prologue GEMM B: " + err; return kp; }
  if (vb.ksplit) { kp.reject = "prologue GEMM B: K-split view"; return kp; }
  if (g.dtype_of(vb.src) != DType::BF16) { kp.reject = "prologue GEMM: B must be bf16"; return kp; }
  for (int m : c.members)
    if (g.prims[m].kind == Kind::Reduce && g.topo_index[m] > g.topo_index[mm]) {
      kp.reject = "prologue GEMM: no epilogue reductions";
      return kp;
    }
  const Shape& C = L.shape;
  const int nbC = (int)C.size() - 2;
  const Shape& as = g.shape_of(L.in[0]);
  const int64_t M = C[nbC], N = C[nbC + 1], K = as.back();
  const int nbB = (int)vb.shape.size() - 2;
  if ((int)as.size() - 2 != nbC || (nbB != 0 && nbB != nbC)) { kp.reject = "prologue GEMM: batch layout"; return kp; }
  if (K % 64 || K > 768) { kp.reject = "prologue GEMM: K % 64 != 0 or K > 768"; return kp; }
  const int64_t b_k = vb.coef[nbB], b_n = vb.coef[nbB + 1];
  const bool b_kmaj = b_k == 1, b_nmaj = !b_kmaj && (b_n == 1 || N == 1);
  if (!(b_kmaj || b_nmaj) || (vb.off * 2) % 16) { kp.reject = "prologue GEMM: B not TMA-able"; return kp; }
  GemmPrologue pro;
  std::vector<Ref> pre{vb.src};
  if (!make_gemm_prologue(g, c, mm, pre, &pro, &err)) { kp.reject = "prologue: " + err; return kp; }
  const int64_t NKA = K / 64;
  const int A_RES = (int)(NKA * 16384);
  int64_t batch = 1;
  for (int b = 0; b < nbC; ++b) batch *= C[b];
  kp.flops = 2.0 * (double)M * (double)N * (double)K * (double)batch;
  for (int BN : {16, 32, 64, 128}) {
    if (BN > 64 && BN / 2 >= N) continue;
    const int CW = BN < 32 ? BN : 32;
    GemmEpilogue ep;
    if (!make_gemm_epilogue(g, c, mm, CW, pro.ext, &ep, &err)) { kp.reject = err; continue; }
    const int B_BYTES = BN * 64 * 2;
    const int budget = 227 * 1024 - A_RES - 1024 - 256;
    const int S = (int)std::min<int64_t>(NKA, budget / B_BYTES);
    if (S < std::min<int64_t>(2, NKA)) { kp.reject = "prologue GEMM: shared memory"; continue; }
    const int smem = A_RES + S * B_BYTES + 1024 + (2 * S + 3) * 8 + 16;
    const int TE = epilogue_lanes(g, c, mm, CW, pro.ext, (int64_t)A_RES + (int64_t)S * B_BYTES, &ep);
    const int tcols = tmem_cols(BN);
    const int64_t Mt = (M + 127) / 128, Nt = (N + BN - 1) / BN;
    const int bmn_box = BN < 64 ? BN : 64;
    const int b_swz_tma = bmn_box == 64 ? 3 : bmn_box == 32 ? 2 : 1;
    const int b_swz_umma = bmn_box == 64 ? 2 : bmn_box == 32 ? 4 : 6;
    const int b_row_bytes = bmn_box * 2;
    TmaDesc db;
    std::vector<int> bb_axes;
    {
      db.tensor = 0;
      db.dtype = 1;
      db.swizzle = 3;
      db.elem_off = vb.off;
      db.rank = 0;
      auto push = [&](int64_t dim, int64_t st, uint32_t box) {
        db.dims[db.rank] = dim; db.strides[db.rank] = st * 2; db.box[db.rank] = box; db.rank++;
      };
      if (b_kmaj) { push(K, 1, 64); push(N, N > 1 ? b_n : K, (uint32_t)BN); }
      else { push(N, 1, (uint32_t)bmn_box); push(K, b_k, 64); db.swizzle = b_swz_tma; }
      bool ok = true;
      for (int b = 0; b < nbB; ++b)
        if (vb.coef[b] != 0 && vb.shape[b] > 1) {
          if (db.rank >= 5) ok = false;
          else { push(vb.shape[b], vb.coef[b], 1); bb_axes.push_back(b); }
        }
      for (int i = 1; i < db.rank; ++i)
        if (db.strides[i] % 16 || db.strides[i] <= 0) ok = false;
      if (!ok) { kp.reject = "prologue GEMM: B strides not TMA-able"; continue; }
    }
    // the A-shaped external operand (e.g. the LayerNorm input) arrives by TMA in the
    // resident A tile's own swizzled layout; the prologue then transforms it in place
    const bool staged = pro.stage_slot >= 0;
    TmaDesc dx;
    std::vector<int> bx_axes;
    if (staged) {
      dx.tensor = pro.stage_slot;
      dx.dtype = 1;
      dx.swizzle = 3;
      dx.elem_off = 0;
      dx.rank = 0;
      auto push = [&](int64_t dim, int64_t st, uint32_t box) {
        dx.dims[dx.rank] = dim; dx.strides[dx.rank] = st * 2; dx.box[dx.rank] = box; dx.rank++;
      };
      push(K, 1, 64);
      push(M, K, 128);
      int64_t st = M * K;
      for (int b = nbC - 1; b >= 0; --b) {
        if (as[b] > 1) {
          if (dx.rank >= 5) { kp.reject = "prologue GEMM: staged operand rank"; break; }
          push(as[b], st, 1);
          bx_axes.push_back(b);
        }
        st *= as[b];
      }
      if (dx.rank > 5 || (dx.rank == 5 && bx_axes.size() + 2 != 5)) continue;
    }
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((b_kmaj ? 0u : 1u) << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    auto coords = [&](const std::string& inner, const std::string& outer) {
      std::string s2 = inner + ", " + outer;
      for (int b : bb_axes) s2 += ", " + ep.batch_vars[b];
      return s2;
    };
    const std::string load = "tma_load_" + std::to_string(db.rank) + "d";
    std::ostringstream k;
    k << "extern \"C\" __global__ void __launch_bounds__(192, 1) KNAME(";
    for (size_t i = 0; i < ep.ext.size(); ++i)
      k << "const " << (g.dtype_of(ep.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
    k << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c) << ", "
      << "const __grid_constant__ TmaMap tmB" << (staged ? ", const __grid_constant__ TmaMap tmX" : "") << ") {\n";
    k << "  typedef " << (numel(C) >= (1LL << 31) ? "long long" : "int") << " idx_t;\n";
    k << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
    k << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
    k << "  unsigned long long* full = (unsigned long long*)(smem + " << A_RES + S * B_BYTES << ");\n";
    k << "  unsigned long long* empty = full + " << S << ";\n";
    k << "  unsigned long long* aready = empty + " << S << ";\n";
    k << "  unsigned long long* accf = aready + 1;\n";
    k << "  unsigned long long* xfull = accf + 1;\n";
    k << "  unsigned* tslot = (unsigned*)(xfull + 1);\n";
    k << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
    k << "  const int tile_m = blockIdx.x * 128, tile_n = blockIdx.y * " << BN << ";\n";
    k << "  int bzl = blockIdx.z;\n";
    for (int b = nbC - 1; b >= 0; --b)
      k << "  const int " << ep.batch_vars[b] << " = bzl % " << C[b] << "; bzl /= " << C[b] << ";\n";
    k << "  (void)bzl;\n";
    // B loads (kb, sb, s in scope)
    std::ostringstream ldb;
    if (b_kmaj) {
      ldb << "      " << load << "(sb, &tmB, full + s, " << coords("kb * 64", "tile_n") << ");\n";
    } else {
      for (int cc = 0; cc < (BN + 63) / 64; ++cc)
        ldb << "      " << load << "(sb + " << cc * 8192 << ", &tmB, full + s, " << coords("tile_n + " + str(cc * 64), "kb * 64")
            << ");\n";
    }
    std::string xc;
    for (int b : bx_axes) xc += ", " + ep.batch_vars[b];
    std::ostringstream ldx;
    if (staged) {
      ldx << "    mbar_expect_tx(xfull, " << A_RES << "u);\n";
      ldx << "    for (int kb = 0; kb < " << NKA << "; ++kb)\n";
      ldx << "      tma_load_" << dx.rank << "d(smem + kb * 16384, &tmX, xfull, kb * 64, tile_m" << xc << ");\n";
    }
    // graph-input operands (weights; the staged LayerNorm input when it is a graph input)
    // are fetched right after barrier init, before the programmatic-dependency wait
    const bool earlyB = vb.src.is_input;
    const bool earlyX = staged && pro.ext[pro.stage_slot].is_input;
    const int64_t PRE = earlyB ? std::min<int64_t>(S, NKA) : 0;
    k << "  if (threadIdx.x == 0) {\n    for (int s = 0; s < " << S
      << "; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }\n"
      << "    mbar_init(aready, 4);\n    mbar_init(accf, 1);\n    mbar_init(xfull, 1);\n    mbar_fence_init();\n"
      << "    tma_prefetch(&tmB);\n" << (staged ? "    tma_prefetch(&tmX);\n" : "");
    if (earlyX) k << ldx.str();
    if (PRE) {
      k << "    for (int s = 0; s < " << PRE << "; ++s) {\n      const int kb = s;\n";
      k << "      mbar_expect_tx(full + s, " << B_BYTES << "u);\n";
      k << "      unsigned char* sb = smem + " << A_RES << " + s * " << B_BYTES << ";\n";
      k << ldb.str() << "    }\n";
    }
    k << "  }\n";
    k << "  if (warp == 5) tc_alloc(tslot, " << tcols << ");\n";
    k << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
    k << "  const unsigned tmem = *tslot;\n";
    k << "  pdl_trigger();\n  pdl_wait();\n";
    k << "  if (warp < 4) {\n";
    // prologue: one warp per A row
    k << "    const unsigned sA = smem_u32(smem);\n    const int tid = lane;\n    const unsigned gmask = 0xffffffffu;\n"
      << "    (void)gmask;\n";
    if (staged) k << "    mbar_wait(xfull, 0);\n";
    k << "    #pragma unroll 1\n    for (int r = warp; r < 128; r += 4) {\n";
    k << "      const int gm = tile_m + r;\n      if (gm >= " << M << ") break;\n";
    k << pro.body;
    k << "    }\n";
    k << "    fence_async_smem();\n    __syncwarp();\n    if (lane == 0) mbar_arrive(aready);\n";
    k << "  } else if (warp == 4 && lane == 0) {\n";
    if (staged && !earlyX) k << ldx.str();
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = 0; kb < " << NKA << "; ++kb) {\n";
    k << "      mbar_wait(empty + s, ph ^ 1u);\n";
    k << "      if (kb >= " << PRE << ") {\n";
    k << "      mbar_expect_tx(full + s, " << B_BYTES << "u);\n";
    k << "      unsigned char* sb = smem + " << A_RES << " + s * " << B_BYTES << ";\n";
    k << ldb.str() << "      }\n";
    k << "      if (++s == " << S << ") { s = 0; ph ^= 1u; }\n    }\n";
    k << "  } else if (warp == 5 && lane == 0) {\n";
    k << "    mbar_wait(aready, 0);\n    tc_fence_after();\n";
    k << "    const unsigned sa0 = smem_u32(smem);\n";
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = 0; kb < " << NKA << "; ++kb) {\n";
    k << "      mbar_wait(full + s, ph);\n      tc_fence_after();\n";
    k << "      const unsigned sa = sa0 + kb * 16384, sb = sa0 + " << A_RES << " + s * " << B_BYTES << ";\n";
    k << "      #pragma unroll\n      for (int k = 0; k < 4; ++k) {\n";
    k << "        const unsigned long long ad = umma_desc(sa + k * 32, 16, 1024);\n";
    if (b_kmaj)
      k << "        const unsigned long long bd = umma_desc(sb + k * 32, 16, 1024);\n";
    else
      k << "        const unsigned long long bd = umma_desc(sb + k * " << 16 * b_row_bytes << ", 8192, " << 8 * b_row_bytes
        << ", " << b_swz_umma << ");\n";
    k << "        tc_mma(tmem, ad, bd, " << idesc << "u, (kb | k) != 0);\n      }\n";
    k << "      tc_commit(empty + s);\n";
    k << "      if (++s == " << S << ") { s = 0; ph ^= 1u; }\n    }\n";
    k << "    tc_commit(accf);\n  }\n";
    k << "  __syncwarp();\n";
    k << "  if (warp < 4) {\n    mbar_wait(accf, 0);\n    __syncwarp();\n    tc_fence_after();\n";
    k << emit_tmem_epilogue(ep, BN, CW, TE, M, N);
    k << "  }\n";
    k << "  tc_fence_before();\n  __syncthreads();\n";
    k << "  if (warp == 5) tc_dealloc(tmem, " << tcols << ");\n}\n";
    KernelVariant kv;
    std::string src = k.str();
    char nm[64];
    std::snprintf(nm, sizeof nm, "korch_pgemm_%016llx", (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + src));
    kv.name = nm;
    src.replace(src.find("KNAME"), 5, kv.name);
    kv.source = src;
    kv.tcgen05 = true;
    kv.block = 192;
    kv.grid = Mt;
    kv.grid_y = Nt;
    kv.grid_z = batch;
    kv.smem = smem;
    kv.tma = {db};
    if (staged) kv.tma.push_back(dx);
    std::ostringstream t;
    t << "gemm-prologue" << (staged ? "-tma" : "") << " BM=128 BN=" << BN << " K=" << K << " stagesB=" << S << " B=" << (b_kmaj ? "K" : "N")
      << "-major M=" << M << " N=" << N << " batch=" << batch << (TE > 1 ? " epi=cl" : "");
    kv.tag = t.str();
    kp.ext = ep.ext;
    kp.bytes = ep.bytes + pro.bytes + 2 * numel(vb.shape);
    kp.variants.push_back(kv);

    // KB5-PC: cluster-shared prologue.  The variant above recomputes the prologue (e.g. a
    // LayerNorm over all 128 rows of the A tile) in every CTA of a tile row, serially on 4
    // warps.  Here a cluster of CN CTAs along N shares the prologue: CTA rank cr TMA-loads
    // only its RP = 128 / CN rows of the staged input, runs the prologue on them (one or
    // two rows per warp on up to 16 prologue warps) and TMA-stores the bf16 rows into the
    // cluster's own copy of A in the kernel's scratch buffer ([Nt / CN][M][K] bf16,
    // L2-resident; clusters never write the same lines); after a cluster barrier the A
    // tile comes back from the scratch either multicast (each CTA loads its slice with
    // .multicast::cluster into all CN CTAs) or per CTA (each CTA loads all 128 rows), so
    // the prologue runs once per row per cluster.  Single-batch GEMMs only.
    for (int CNM : {8, 4, -8, -4}) {
      const int CN = CNM < 0 ? -CNM : CNM;
      const bool MC = CNM > 0;                   // multicast the slices, else every CTA loads all rows
      const int RP = 128 / CN;
      const int PW = RP < 16 ? RP : 16;          // prologue warps (one or two rows each)
      const int NT = 32 * (PW + 2);              // + the TMA warp PW and the MMA warp PW + 1
      if (!staged || batch != 1 || !bx_axes.empty() || dx.rank != 2 || Nt % CN || RP % 8) continue;
      TmaDesc dxs = dx, dsc = dx;
      dxs.box[1] = (uint32_t)RP;
      dsc.tensor = -3;
      dsc.elem_off = 0;
      dsc.box[1] = (uint32_t)RP;
      // one scratch copy of the A tile row per cluster (clusters never write the same lines)
      const int64_t NCL = Nt / CN;
      dsc.rank = 3;
      dsc.dims[2] = NCL;
      dsc.strides[2] = M * K * 2;
      dsc.box[2] = 1;
      std::ostringstream q;
      q << "static __device__ __forceinline__ void tma_load_3d_mc(void* dst, const TmaMap* m, unsigned long long* bar, int c0,\n"
           "                                                      int c1, unsigned short mask, int c2) {\n"
           "  asm volatile(\"cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster\"\n"
           "               \" [%0], [%1, {%3, %4, %6}], [%2], %5;\" ::\"r\"(smem_u32(dst)), \"l\"((unsigned long long)m),\n"
           "               \"r\"(smem_u32(bar)), \"r\"(c0), \"r\"(c1), \"h\"(mask), \"r\"(c2) : \"memory\");\n}\n"
           "static __device__ __forceinline__ void tma_store_3d(const TmaMap* m, const void* src, int c0, int c1, int c2) {\n"
           "  asm volatile(\"cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\" ::\"l\"(\n"
           "               (unsigned long long)m), \"r\"(smem_u32(src)), \"r\"(c0), \"r\"(c1), \"r\"(c2) : \"memory\");\n}\n";
      q << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", 1) KNAME(";
      for (size_t i = 0; i < ep.ext.size(); ++i)
        q << "const " << (g.dtype_of(ep.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
      q << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c)
        << ", bf16_t* __restrict__ scratch, const __grid_constant__ TmaMap tmB, const __grid_constant__ TmaMap tmX, "
           "const __grid_constant__ TmaMap tmS) {\n";
      q << "  typedef " << (numel(C) >= (1LL << 31) ? "long long" : "int") << " idx_t;\n  (void)scratch;\n";
      q << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
      q << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
      q << "  unsigned long long* full = (unsigned long long*)(smem + " << A_RES + S * B_BYTES << ");\n";
      q << "  unsigned long long* empty = full + " << S << ";\n";
      q << "  unsigned long long* afull = empty + " << S << ";\n";
      q << "  unsigned long long* accf = afull + 1;\n";
      q << "  unsigned long long* xfull = accf + 1;\n";
      q << "  unsigned* tslot = (unsigned*)(xfull + 1);\n";
      q << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
      q << "  const int tile_n = blockIdx.x * " << BN << ", tile_m = blockIdx.y * 128;\n";
      q << "  unsigned cr;\n  asm volatile(\"mov.u32 %0, %%cluster_ctarank;\" : \"=r\"(cr));\n";
      q << "  const int row0 = (int)cr * " << RP << ", cl = (int)(blockIdx.x / " << CN << ");\n";
      q << "  int bzl = blockIdx.z;\n";
      for (int b = nbC - 1; b >= 0; --b)
        q << "  const int " << ep.batch_vars[b] << " = bzl % " << C[b] << "; bzl /= " << C[b] << ";\n";
      q << "  (void)bzl;\n";
      std::ostringstream ldxs;
      ldxs << "    mbar_expect_tx(xfull, " << RP * K * 2 << "u);\n";
      ldxs << "    for (int kb = 0; kb < " << NKA << "; ++kb)\n";
      ldxs << "      tma_load_2d(smem + kb * 16384 + row0 * 128, &tmX, xfull, kb * 64, tile_m + row0);\n";
      q << "  if (threadIdx.x == 0) {\n    for (int s = 0; s < " << S
        << "; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }\n"
        << "    mbar_init(afull, 1);\n    mbar_init(accf, 1);\n    mbar_init(xfull, 1);\n    mbar_fence_init();\n"
        << "    tma_prefetch(&tmB);\n    tma_prefetch(&tmX);\n    tma_prefetch(&tmS);\n";
      // armed before the cluster barrier below, so no peer's multicast can precede it
      q << "    mbar_expect_tx(afull, " << A_RES << "u);\n";
      if (earlyX) q << ldxs.str();
      if (PRE) {
        q << "    for (int s = 0; s < " << PRE << "; ++s) {\n      const int kb = s;\n";
        q << "      mbar_expect_tx(full + s, " << B_BYTES << "u);\n";
        q << "      unsigned char* sb = smem + " << A_RES << " + s * " << B_BYTES << ";\n";
        q << ldb.str() << "    }\n";
      }
      q << "  }\n";
      q << "  if (warp == " << PW + 1 << ") tc_alloc(tslot, " << tcols << ");\n";
      q << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
      q << "  const unsigned tmem = *tslot;\n";
      q << "  asm volatile(\"barrier.cluster.arrive.relaxed.aligned;\\nbarrier.cluster.wait.aligned;\" ::: \"memory\");"
           "  // every CTA's barriers are initialised and armed\n";
      q << "  pdl_trigger();\n  pdl_wait();\n";
      q << "  if (warp < " << PW << ") {\n";
      if (!earlyX) q << "    if (threadIdx.x == 0) {\n" << ldxs.str() << "    }\n";
      q << "    const unsigned sA = smem_u32(smem);\n    const int tid = lane;\n    const unsigned gmask = 0xffffffffu;\n"
        << "    (void)gmask;\n";
      q << "    mbar_wait(xfull, 0);\n";
      q << "    #pragma unroll 1\n    for (int r = row0 + warp; r < row0 + " << RP << "; r += " << PW << ") {\n";
      q << "      const int gm = tile_m + r;\n      if (gm >= " << M << ") break;\n";
      q << pro.body;
      q << "    }\n";
      // the prologue's st.shared -> async proxy; then one thread stores the slice to the
      // scratch and waits for the bulk writes to complete before the cluster barrier
      q << "    fence_async_smem();\n    named_bar_sync(1, " << 32 * PW << ");\n";
      q << "    if (threadIdx.x == 0) {\n";
      q << "      for (int kb = 0; kb < " << NKA << "; ++kb) tma_store_3d(&tmS, smem + kb * 16384 + row0 * 128, kb * 64, tile_m + row0, cl);\n";
      q << "      asm volatile(\"cp.async.bulk.commit_group;\" ::: \"memory\");\n";
      q << "      asm volatile(\"cp.async.bulk.wait_group 0;\" ::: \"memory\");\n";
      q << "      asm volatile(\"fence.proxy.async.global;\" ::: \"memory\");\n    }\n";
      q << "    __syncwarp();\n  }\n";
      q << "  cluster_sync();  // every slice of the A tile is in the scratch\n";
      q << "  if (warp == " << PW << " && lane == 0) {\n";
      q << "    asm volatile(\"fence.proxy.async.global;\" ::: \"memory\");\n";
      if (MC) {
        q << "    for (int kb = 0; kb < " << NKA << "; ++kb)\n";
        q << "      tma_load_3d_mc(smem + kb * 16384 + row0 * 128, &tmS, afull, kb * 64, tile_m + row0, (unsigned short)"
          << ((1 << CN) - 1) << ", cl);\n";
      } else {
        q << "    for (int kb = 0; kb < " << NKA << "; ++kb)\n";
        q << "      for (int c = 0; c < " << CN << "; ++c)\n";
        q << "        tma_load_3d(smem + kb * 16384 + c * " << RP * 128 << ", &tmS, afull, kb * 64, tile_m + c * " << RP << ", cl);\n";
      }
      q << "    int s = 0; unsigned ph = 0;\n";
      q << "    for (int kb = 0; kb < " << NKA << "; ++kb) {\n";
      q << "      mbar_wait(empty + s, ph ^ 1u);\n";
      q << "      if (kb >= " << PRE << ") {\n";
      q << "      mbar_expect_tx(full + s, " << B_BYTES << "u);\n";
      q << "      unsigned char* sb = smem + " << A_RES << " + s * " << B_BYTES << ";\n";
      q << ldb.str() << "      }\n";
      q << "      if (++s == " << S << ") { s = 0; ph ^= 1u; }\n    }\n";
      q << "  } else if (warp == " << PW + 1 << " && lane == 0) {\n";
      q << "    mbar_wait(afull, 0);\n    tc_fence_after();\n";
      q << "    const unsigned sa0 = smem_u32(smem);\n";
      q << "    int s = 0; unsigned ph = 0;\n";
      q << "    for (int kb = 0; kb < " << NKA << "; ++kb) {\n";
      q << "      mbar_wait(full + s, ph);\n      tc_fence_after();\n";
      q << "      const unsigned sa = sa0 + kb * 16384, sb = sa0 + " << A_RES << " + s * " << B_BYTES << ";\n";
      q << "      #pragma unroll\n      for (int k = 0; k < 4; ++k) {\n";
      q << "        const unsigned long long ad = umma_desc(sa + k * 32, 16, 1024);\n";
      if (b_kmaj)
        q << "        const unsigned long long bd = umma_desc(sb + k * 32, 16, 1024);\n";
      else
        q << "        const unsigned long long bd = umma_desc(sb + k * " << 16 * b_row_bytes << ", 8192, " << 8 * b_row_bytes
          << ", " << b_swz_umma << ");\n";
      q << "        tc_mma(tmem, ad, bd, " << idesc << "u, (kb | k) != 0);\n      }\n";
      q << "      tc_commit(empty + s);\n";
      q << "      if (++s == " << S << ") { s = 0; ph ^= 1u; }\n    }\n";
      q << "    tc_commit(accf);\n  }\n";
      q << "  __syncwarp();\n";
      q << "  if (warp < 4) {\n    mbar_wait(accf, 0);\n    __syncwarp();\n    tc_fence_after();\n";
      q << emit_tmem_epilogue(ep, BN, CW, TE, M, N);
      q << "  }\n";
      q << "  tc_fence_before();\n  __syncthreads();\n";
      q << "  if (warp == " << PW + 1 << ") tc_dealloc(tmem, " << tcols << ");\n}\n";
      KernelVariant kc;
      std::string s2 = q.str();
      std::snprintf(nm, sizeof nm, "korch_pgemm_%016llx", (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + s2));
      kc.name = nm;
      s2.replace(s2.find("KNAME"), 5, kc.name);
      kc.source = s2;
      kc.tcgen05 = true;
      kc.block = NT;
      kc.grid = Nt;
      kc.grid_y = Mt;
      kc.grid_z = 1;
      kc.cluster = CN;
      kc.smem = smem;
      kc.scratch_bytes = NCL * M * K * 2;
      kc.tma = {db, dxs, dsc};
      kc.tag = t.str() + " cluster-prologue CN=" + std::to_string(CN) + " PW=" + std::to_string(PW) +
               (MC ? " A=multicast" : " A=per-CTA");
      kp.variants.push_back(kc);
    }
  }
  if (!kp.variants.empty()) {
    kp.klass = KORCH_CLASS_GEMM;
    kp.reject.clear();
  }
  return kp;
}

KernelPlan generate_gemm(const Graph& g, const Candidate& c) {
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  int mm = -1;
  for (int m : c.members)
    if (g.is_dense_linear(m)) mm = m;
  const Prim& L = g.prims[mm];
  if (L.kind == Kind::Conv2d) return generate_conv_gemm(g, c, mm);
  std::set<int> mem(c.members.begin(), c.members.end());
  View va, vb;
  std::set<int> chain;
  std::string err;
  {
    // A computed in the kernel (not a view of an external tensor): the prologue GEMM
    View t;
    std::set<int> ch;
    std::string e2;
    const Ref& a = L.in[0];
    if (!a.is_input && mem.count(a.id) && !operand_view(g, mem, L, 0, &t, &ch, &e2)) return generate_prologue_gemm(g, c, mm);
  }
  if (!operand_view(g, mem, L, 0, &va, &chain, &err) || !operand_view(g, mem, L, 1, &vb, &chain, &err)) {
    kp.reject = err;
    return kp;
  }
  // every member upstream of L must be part of an operand view chain
  {
    std::vector<int> stack{mm};
    std::set<int> anc;
    while (!stack.empty()) {
      int v = stack.back();
      stack.pop_back();
      for (int p : g.preds[v])
        if (mem.count(p) && !anc.count(p)) {
          anc.insert(p);
          stack.push_back(p);
        }
    }
    for (int a : anc)
      if (!chain.count(a)) {
        kp.reject = "computation upstream of the linear primitive (not a view)";
        return kp;
      }
  }
  if (g.dtype_of(va.src) != DType::BF16 || g.dtype_of(vb.src) != DType::BF16) {
    kp.reject = "GEMM operands must be bf16 (tcgen05 kind::f16)";
    return kp;
  }
  const Shape& C = L.shape;
  int nbC = (int)C.size() - 2;
  int64_t M = C[nbC], N = C[nbC + 1], K = va.shape.back();
  int nbA = (int)va.shape.size() - 2, nbB = (int)vb.shape.size() - 2;
  if (nbA != nbC || (nbB != 0 && nbB != nbC)) {
    kp.reject = "unsupported batch broadcast";
    return kp;
  }
  // majorness
  int64_t a_m = va.coef[nbA], a_k = va.coef[nbA + 1], b_k = vb.coef[nbB], b_n = vb.coef[nbB + 1];
  bool a_kmaj = a_k == 1 || K == 1, a_mmaj = !a_kmaj && (a_m == 1 || M == 1);
  bool b_kmaj = b_k == 1 || K == 1, b_nmaj = !b_kmaj && (b_n == 1 || N == 1);
  if (!(a_kmaj || a_mmaj) || !(b_kmaj || b_nmaj)) {
    kp.reject = "operand has no unit-stride axis for TMA";
    return kp;
  }
  if ((va.off * 2) % 16 || (vb.off * 2) % 16) {
    kp.reject = "operand view offset not 16-byte aligned";
    return kp;
  }
  if ((va.ksplit && (va.ksplit % 64 || !a_kmaj || K == 1)) || (vb.ksplit && (vb.ksplit % 64 || K == 1))) {
    kp.reject = "K-split operand view needs 64-aligned splits (and a K-major A)";
    return kp;
  }

  auto build_desc = [&](const View& v, int ext_idx, int64_t inner_dim, int64_t outer_dim, int64_t outer_coef,
                        uint32_t inner_box, uint32_t outer_box, int nbatch, std::vector<int>* batch_axes,
                        TmaDesc* d) -> bool {
    d->tensor = ext_idx;
    d->dtype = 1;
    d->swizzle = 3;
    d->elem_off = v.off;
    d->rank = 0;
    auto push = [&](int64_t dim, int64_t stride_el, uint32_t box) {
      d->dims[d->rank] = dim;
      d->strides[d->rank] = stride_el * 2;
      d->box[d->rank] = box;
      d->rank++;
    };
    // K-split views: the K dimension (inner when K-major, outer otherwise) becomes
    // (k % D) with its own stride plus a (k / D) dimension right after the outer one
    const bool k_inner = inner_box == 64 && v.ksplit && (&v == &va ? a_kmaj : b_kmaj);
    const int64_t D = v.ksplit;
    push(k_inner ? D : inner_dim, 1, inner_box);
    if (D && !k_inner) push(D, outer_coef, outer_box);
    else push(outer_dim, outer_dim > 1 ? outer_coef : (outer_coef ? outer_coef : inner_dim), outer_box);
    if (D) push(K / D, v.kout, 1);
    for (int b = 0; b < nbatch; ++b)
      if (v.coef[b] != 0 && v.shape[b] > 1) {
        if (d->rank >= 5) return false;
        push(v.shape[b], v.coef[b], 1);
        batch_axes->push_back(b);
      }
    for (int i = 1; i < d->rank; ++i)
      if (d->strides[i] % 16 || d->strides[i] <= 0 || d->strides[i] >= (1LL << 40)) return false;
    return true;
  };

  bool has_reduce = false;
  for (int m : c.members)
    if (g.prims[m].kind == Kind::Reduce) has_reduce = true;
  if (has_reduce && (N % 32 || N > 256)) {
    kp.reject = "in-tile row reduction needs N % 32 == 0 and N <= 256";
    return kp;
  }
  std::vector<Ref> pre{va.src, vb.src};
  GemmEpilogue ep;
  if (!make_gemm_epilogue(g, c, mm, has_reduce ? (int)N : 32, pre, &ep, &err)) {
    kp.reject = err;
    return kp;
  }
  int slotA = 0, slotB = (va.src.is_input == vb.src.is_input && va.src.id == vb.src.id) ? 0 : 1;
  kp.ext = ep.ext;
  int64_t batch = 1;
  for (int b = 0; b < nbC; ++b) batch *= C[b];
  kp.flops = 2.0 * (double)M * (double)N * (double)K * (double)batch;
  int64_t a_el = numel(va.shape), b_el = numel(vb.shape);
  kp.bytes = ep.bytes + 2 * (a_el + b_el);

  // Launch configurations (the profiler keeps the fastest):
  //  * tile width BN: small BN spreads a skinny (small-M, weight-streaming) GEMM over more
  //    SMs, large BN maximises operand reuse;
  //  * split-K (KS > 1) for grids far smaller than the 148 SMs: a cluster of KS CTAs
  //    accumulates the K-slices of one tile in their TMEMs and reduces them through
  //    distributed shared memory (see the KS > 1 epilogue below).
  struct Cfg { int bn, ks; bool persist = false; int ew = 1; };
  std::vector<Cfg> cfgs;
  const int64_t NKt = (K + 63) / 64;
  const int64_t Mt = (M + 127) / 128;
  if (has_reduce) {
    cfgs.push_back({(int)N, 1});  // in-tile row reduction: one tile spans the whole row
  } else {
    for (int bn : {16, 32, 64, 128, 256})
      if (bn <= 64 || bn / 2 < N) cfgs.push_back({bn, 1});
    for (int bn : {32, 64, 128})
      for (int ks : {2, 4, 8}) {
        int64_t tiles = Mt * ((N + bn - 1) / bn) * batch;
        if (bn > 64 && bn / 2 >= N) continue;
        if (NKt % ks || tiles >= 148 || tiles * ks > 2 * 148 || N % 32 || N < bn) continue;
        cfgs.push_back({bn, ks});
      }
    // persistent tile loop with double-buffered TMEM accumulators (large grids only)
    for (int bn : {128, 256}) {
      const int64_t tiles = Mt * ((N + bn - 1) / bn) * batch;
      if (tiles >= 2 * 148 && bn / 2 < N) {
        cfgs.push_back({bn, 1, true, 1});
        cfgs.push_back({bn, 1, true, 2});  // two epilogue warps per TMEM lane quarter
      }
    }
  }
  bool gather_fallback = false;
  for (const Cfg& cf : cfgs) {
    const int BN = cf.bn, KS = cf.ks;
    // epilogue chunk (TMEM columns per pass); the whole row when reducing
    const int CW = has_reduce ? BN : (BN < 32 ? BN : 32);
    GemmEpilogue epv;
    if (!make_gemm_epilogue(g, c, mm, CW, pre, &epv, &err)) continue;
    TmaDesc da, db;
    std::vector<int> ba_axes, bb_axes;
    // MN-major B narrower than a 128B swizzle atom uses the 64B / 32B swizzle modes
    const int bmn_box = BN < 64 ? BN : 64;
    const int b_swz_tma = bmn_box == 64 ? 3 : bmn_box == 32 ? 2 : 1;       // CUtensorMapSwizzle
    const int b_swz_umma = bmn_box == 64 ? 2 : bmn_box == 32 ? 4 : 6;      // UMMA layout type
    const int b_row_bytes = bmn_box * 2;                                    // one K row of a B atom
    bool ok = a_kmaj ? build_desc(va, slotA, K, M, a_m, 64, 128, nbA, &ba_axes, &da)
                     : build_desc(va, slotA, M, K, a_k, 64, 64, nbA, &ba_axes, &da);
    ok = ok && (b_kmaj ? build_desc(vb, slotB, K, N, b_n, 64, (uint32_t)BN, nbB, &bb_axes, &db)
                       : build_desc(vb, slotB, N, K, b_k, (uint32_t)bmn_box, 64, nbB, &bb_axes, &db));
    if (!ok) {
      kp.reject = "operand strides not expressible as a TMA tensor map";
      gather_fallback = true;
      continue;
    }
    if (!b_kmaj) db.swizzle = b_swz_tma;
    if (cf.persist) {
      // KB5-persistent: one CTA per SM walks the tiles t = blockIdx.x, +gridDim.x, ...
      // warp 0 = TMA producer (ring of S stages shared by consecutive tiles), warp 1 = MMA
      // issuer into one of two TMEM accumulators (2 x BN columns), warps 2-5 = epilogue
      // (TMEM lane quarter = warp % 4), which drains tile i's accumulator while the MMA
      // warp fills the other one with tile i+1: the epilogue and the next tile's operand
      // stream overlap instead of serialising per CTA.
      const int A_BYTES = 128 * 64 * 2, B_BYTES = BN * 64 * 2, STAGE = A_BYTES + B_BYTES;
      const int64_t NK = NKt;
      GemmEpilogue pe = epv;
      const int TE = epilogue_lanes(g, c, mm, CW, pre, 1 << 30, &pe, 0);
      const int EW = cf.ew, BNh = BN / EW;     // epilogue warp groups, columns each drains
      if (BNh % CW) continue;
      const int STG = TE > 1 ? EW * stage_bytes(CW) : 0;
      const int S = (int)std::min<int64_t>(NK < 2 ? 2 : NK, (220 * 1024 - STG - 2048) / STAGE);
      if (S < 2) continue;
      const int64_t STG_OFF = (int64_t)S * STAGE, BAR_OFF = STG_OFF + STG;
      const int smem = (int)BAR_OFF + (2 * S + 4) * 8 + 16 + 1024;
      const int64_t Nt = (N + BN - 1) / BN, NT = Mt * Nt * batch;
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((a_kmaj ? 0u : 1u) << 15) | ((b_kmaj ? 0u : 1u) << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      auto coords = [&](std::string inner, std::string outer, const std::vector<int>& baxes, const View& v,
                        bool k_inner) {
        std::string extra;
        if (v.ksplit) {
          std::string& kc = k_inner ? inner : outer;
          extra = ", (" + kc + ") / " + str(v.ksplit);
          kc = "(" + kc + ") % " + str(v.ksplit);
        }
        std::string r = inner + ", " + outer + extra;
        for (int b : baxes) r += ", " + pe.batch_vars[b];
        return r;
      };
      auto load = [&](int rank) { return "tma_load_" + std::to_string(rank) + "d"; };
      std::ostringstream decode;
      decode << "      int tt = t;\n      const int tile_m = (tt % " << Mt << ") * 128; tt /= " << Mt << ";\n"
             << "      const int tile_n = (tt % " << Nt << ") * " << BN << "; tt /= " << Nt << ";\n"
             << "      int bzl = tt;\n";
      for (int b = nbC - 1; b >= 0; --b)
        decode << "      const int " << pe.batch_vars[b] << " = bzl % " << C[b] << "; bzl /= " << C[b] << ";\n";
      decode << "      (void)bzl; (void)tile_m; (void)tile_n;\n";
      std::ostringstream k;
      k << "extern \"C\" __global__ void __launch_bounds__(" << 64 + 128 * EW << ", 1) KNAME(";
      for (size_t i = 0; i < kp.ext.size(); ++i)
        k << "const " << (g.dtype_of(kp.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
      k << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c) << ", ";
      k << "const __grid_constant__ TmaMap tmA, const __grid_constant__ TmaMap tmB) {\n";
      k << "  typedef int idx_t;\n";
      k << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
      k << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
      k << "  unsigned long long* full = (unsigned long long*)(smem + " << BAR_OFF << ");\n";
      k << "  unsigned long long* empty = full + " << S << ";\n";
      k << "  unsigned long long* accfull = empty + " << S << ";\n";
      k << "  unsigned long long* accempty = accfull + 2;\n";
      k << "  unsigned* tslot = (unsigned*)(accempty + 2);\n";
      k << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
      k << "  if (threadIdx.x == 0) {\n    for (int s = 0; s < " << S
        << "; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }\n"
        << "    mbar_init(accfull, 1); mbar_init(accfull + 1, 1); mbar_init(accempty, " << 128 * EW << "); mbar_init(accempty + 1, " << 128 * EW << ");\n"
        << "    mbar_fence_init();\n    tma_prefetch(&tmA);\n    tma_prefetch(&tmB);\n  }\n";
      k << "  if (warp == 1) tc_alloc(tslot, " << 2 * BN << ");\n";
      k << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
      k << "  const unsigned tmem = *tslot;\n";
      k << "  pdl_trigger();\n  pdl_wait();\n";
      // producer
      k << "  if (warp == 0 && lane == 0) {\n    int s = 0; unsigned ph = 0;\n";
      k << "    for (int t = blockIdx.x; t < " << NT << "; t += gridDim.x) {\n" << decode.str();
      k << "      for (int kb = 0; kb < " << NK << "; ++kb) {\n";
      k << "        mbar_wait(empty + s, ph ^ 1u);\n";
      k << "        mbar_expect_tx(full + s, " << STAGE << "u);\n";
      k << "        unsigned char* sa = smem + s * " << STAGE << ";\n        unsigned char* sb = sa + " << A_BYTES << ";\n";
      if (a_kmaj) {
        k << "        " << load(da.rank) << "(sa, &tmA, full + s, " << coords("kb * 64", "tile_m", ba_axes, va, true) << ");\n";
      } else {
        for (int cc = 0; cc < 2; ++cc)
          k << "        " << load(da.rank) << "(sa + " << cc * 8192 << ", &tmA, full + s, "
            << coords("tile_m + " + str(cc * 64), "kb * 64", ba_axes, va, false) << ");\n";
      }
      if (b_kmaj) {
        k << "        " << load(db.rank) << "(sb, &tmB, full + s, " << coords("kb * 64", "tile_n", bb_axes, vb, true) << ");\n";
      } else {
        for (int cc = 0; cc < (BN + 63) / 64; ++cc)
          k << "        " << load(db.rank) << "(sb + " << cc * 8192 << ", &tmB, full + s, "
            << coords("tile_n + " + str(cc * 64), "kb * 64", bb_axes, vb, false) << ");\n";
      }
      k << "        if (++s == " << S << ") { s = 0; ph ^= 1u; }\n      }\n    }\n";
      // MMA issuer
      k << "  } else if (warp == 1 && lane == 0) {\n    int s = 0; unsigned ph = 0; int it = 0;\n";
      k << "    for (int t = blockIdx.x; t < " << NT << "; t += gridDim.x, ++it) {\n";
      k << "      const int buf = it & 1;\n      const unsigned use = (unsigned)(it >> 1);\n";
      k << "      mbar_wait(accempty + buf, (use & 1u) ^ 1u);\n      tc_fence_after();\n";
      k << "      const unsigned acc_t = tmem + (unsigned)(buf * " << BN << ");\n";
      k << "      for (int kb = 0; kb < " << NK << "; ++kb) {\n";
      k << "        mbar_wait(full + s, ph);\n        tc_fence_after();\n";
      k << "        const unsigned sa = smem_u32(smem + s * " << STAGE << "), sb = sa + " << A_BYTES << ";\n";
      k << "        #pragma unroll\n        for (int k = 0; k < 4; ++k) {\n";
      k << "          const unsigned long long ad = umma_desc(sa + " << (a_kmaj ? "k * 32" : "k * 2048") << ", "
        << (a_kmaj ? 16 : 8192) << ", 1024);\n";
      if (b_kmaj)
        k << "          const unsigned long long bd = umma_desc(sb + k * 32, 16, 1024);\n";
      else
        k << "          const unsigned long long bd = umma_desc(sb + k * " << 16 * b_row_bytes << ", 8192, "
          << 8 * b_row_bytes << ", " << b_swz_umma << ");\n";
      k << "          tc_mma(acc_t, ad, bd, " << idesc << "u, (kb | k) != 0);\n        }\n";
      k << "        tc_commit(empty + s);\n";
      k << "        if (++s == " << S << ") { s = 0; ph ^= 1u; }\n      }\n";
      k << "      tc_commit(accfull + buf);\n    }\n";
      // epilogue warps 2-5
      k << "  } else if (warp >= 2) {\n    const int q = warp & 3, h = (warp - 2) / 4;\n    (void)h;\n    int it = 0;\n";
      k << "    for (int t = blockIdx.x; t < " << NT << "; t += gridDim.x, ++it) {\n";
      k << "      const int buf = it & 1;\n      const unsigned use = (unsigned)(it >> 1);\n" << decode.str();
      k << "      mbar_wait(accfull + buf, use & 1u);\n      __syncwarp();\n      tc_fence_after();\n";
      k << "      const unsigned tmem_b = tmem + (unsigned)(buf * " << BN << ");\n";
      if (EW == 1) {
        k << emit_tmem_epilogue(pe, BN, CW, TE, M, N, "tmem_b", "q", "smem + " + str(STG_OFF));
      } else {  // warp group h drains columns [h * BNh, (h + 1) * BNh) of the tile
        k << "      {\n      const int tile_n_base = tile_n;\n      {\n      const int tile_n = tile_n_base + h * " << BNh << ";\n";
        k << emit_tmem_epilogue(pe, BNh, CW, TE, M, N, "(tmem_b + (unsigned)(h * " + str(BNh) + "))", "q",
                                "smem + " + str(STG_OFF) + " + h * " + str(stage_bytes(CW)));
        k << "      }\n      }\n";
      }
      k << "      tc_fence_before();\n      mbar_arrive(accempty + buf);\n    }\n  }\n";
      k << "  tc_fence_before();\n  __syncthreads();\n";
      k << "  if (warp == 1) tc_dealloc(tmem, " << 2 * BN << ");\n}\n";
      KernelVariant kv;
      std::string src = k.str();
      char nm[64];
      std::snprintf(nm, sizeof nm, "korch_gemm_%016llx",
                    (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + src));
      kv.name = nm;
      src.replace(src.find("KNAME"), 5, kv.name);
      kv.source = src;
      kv.tcgen05 = true;
      kv.block = 64 + 128 * EW;
      kv.grid = std::min<int64_t>(NT, 148);
      kv.grid_y = 1;
      kv.grid_z = 1;
      kv.smem = smem;
      kv.tma = {da, db};
      std::ostringstream t;
      t << "gemm-persistent BM=128 BN=" << BN << " BK=64 stages=" << S << " A=" << (a_kmaj ? "K" : "M") << "-major B="
        << (b_kmaj ? "K" : "N") << "-major M=" << M << " N=" << N << " K=" << K << " batch=" << batch
        << (TE > 1 ? " epi=cl" : "") << (EW > 1 ? " epi-warps=8" : "");
      kv.tag = t.str();
      kp.variants.push_back(kv);
      continue;
    }
    // an MN-major B tile arrives as 64-column TMA boxes: BN = 96 / 160 / 224 (in-tile row
    // reductions over N) occupy ceil(BN / 64) whole boxes in shared memory
    const int A_BYTES = 128 * 64 * 2, B_BYTES = (b_kmaj || BN < 64 ? BN : (BN + 63) / 64 * 64) * 64 * 2, STAGE = A_BYTES + B_BYTES;
    const int64_t NK = NKt / KS;  // K-blocks per CTA
    // Pipeline depth: keep as many K-blocks in flight as shared memory allows (up to all
    // of them) -- small-M GEMMs are bound by TMA round-trip latency, not bandwidth.
    int S = (int)std::max<int64_t>(2, std::min<int64_t>(NK, (200 * 1024) / STAGE));
    // Epilogue mapping.  KS == 1: column-lane staging unless rows are contiguous or the
    // epilogue reduces rows.  KS > 1 (cluster split-K): the owner CTA of a row block runs
    // the epilogue over [RO x BN] with T = BN / 8 lanes per row, straight from the
    // DSMEM-reduced partial sums.
    // KS == 1 column-lane epilogues stage full-tile affine side inputs (residuals) by TMA
    // into shared memory during the main loop (EpiSide): the epilogue then reads them
    // from shared memory instead of waiting on one global round trip per pass.
    const int TE = has_reduce ? 1
                   : KS > 1   ? BN / 8
                              : epilogue_lanes(g, c, mm, CW, pre, (int64_t)S * STAGE, &epv, BN <= 256 ? BN : 0);
    if (KS > 1) {
      GemmEpilogue e2;
      if (!make_gemm_epilogue(g, c, mm, BN, pre, &e2, &err, -1, TE) || e2.ext.size() != epv.ext.size()) continue;
      epv = e2;
    }
    std::vector<int64_t> side_off;
    int64_t side_bytes = 0;
    for (auto& sd : epv.sides) {
      side_off.push_back(side_bytes);
      side_bytes += ((int64_t)128 * BN * (sd.dtype ? 2 : 4) + 1023) / 1024 * 1024;
    }
    if (side_bytes) {
      const int S2 = (int)std::max<int64_t>(2, std::min<int64_t>(NK, (200 * 1024 - side_bytes) / STAGE));
      if ((int64_t)S2 * STAGE + side_bytes > 208 * 1024) {  // no room: plain global side reads
        GemmEpilogue e2;
        if (!make_gemm_epilogue(g, c, mm, CW, pre, &e2, &err, -1, TE) || e2.ext.size() != epv.ext.size()) continue;
        epv = e2;
        side_off.clear();
        side_bytes = 0;
      } else {
        S = S2;
      }
    }
    const GemmEpilogue& ep = epv;
    const int RO = 128 / KS, PB = BN + 4;                  // rows owned per CTA, receive pitch (floats)
    const int64_t recv_bytes = KS > 1 ? (int64_t)128 * PB * 4 : 0;
    // split-K receive buffer: its own region (barrier-free reduction, emit_dsmem_splitk_async)
    // when shared memory allows, else aliasing the idle operand ring (emit_dsmem_splitk)
    const bool rasync = KS > 1 && (int64_t)S * STAGE + recv_bytes + side_bytes + 1024 + (2 * S + 3) * 8 + 16 <= 227 * 1024;
    const int64_t RECV_OFF = rasync ? (int64_t)S * STAGE : 0;
    const int64_t REG0 = rasync ? (int64_t)S * STAGE + recv_bytes : std::max<int64_t>((int64_t)S * STAGE, recv_bytes);
    const int64_t REG = REG0 + side_bytes;                 // ring (| DSMEM receive) | side tiles
    std::vector<TmaDesc> sdesc;
    std::vector<std::vector<int>> sd_axes;
    bool side_ok = true;
    for (auto& sd : ep.sides) {
      TmaDesc d;
      d.tensor = sd.slot;
      d.dtype = sd.dtype;
      d.swizzle = 0;
      d.elem_off = sd.off;
      const int esz = sd.dtype ? 2 : 4;
      auto push = [&](int64_t dim, int64_t st_el, uint32_t box) {
        d.dims[d.rank] = dim; d.strides[d.rank] = st_el * esz; d.box[d.rank] = box; d.rank++;
      };
      push(N, 1, (uint32_t)BN);
      push(M, sd.sm, 128);
      std::vector<int> ax;
      for (int b = 0; b < nbC; ++b)
        if (sd.bcoef[b] != 0 && C[b] > 1) {
          if (d.rank >= 5) side_ok = false;
          else { push(C[b], sd.bcoef[b], 1); ax.push_back(b); }
        }
      for (int i = 1; i < d.rank; ++i)
        if (d.strides[i] % 16 || d.strides[i] <= 0 || d.strides[i] >= (1LL << 40)) side_ok = false;
      sdesc.push_back(d);
      sd_axes.push_back(ax);
    }
    if (!side_ok) continue;
    if (REG + 1024 + (2 * S + 3) * 8 + 16 > 227 * 1024) continue;
    const int smem = (int)REG + 1024 + (2 * S + 3) * 8 + 16;
    const int tcols = tmem_cols(BN);
    const int64_t Nt = (N + BN - 1) / BN;
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((a_kmaj ? 0u : 1u) << 15) | ((b_kmaj ? 0u : 1u) << 16) |
                     ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    // coordinates of a load: K-split views address k as (k % D, .., k / D)
    auto coords = [&](std::string inner, std::string outer, const std::vector<int>& baxes, const View& v,
                      bool k_inner) {
      std::string extra;
      if (v.ksplit) {
        std::string& kc = k_inner ? inner : outer;
        extra = ", (" + kc + ") / " + str(v.ksplit);
        kc = "(" + kc + ") % " + str(v.ksplit);
      }
      std::string s = inner + ", " + outer + extra;
      for (int b : baxes) s += ", " + ep.batch_vars[b];
      return s;
    };
    auto load = [&](int rank) { return "tma_load_" + std::to_string(rank) + "d"; };
    std::ostringstream k;
    k << "extern \"C\" __global__ void __launch_bounds__(128, 1) KNAME(";
    for (size_t i = 0; i < kp.ext.size(); ++i)
      k << "const " << (g.dtype_of(kp.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
    k << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c) << ", ";
    k << "const __grid_constant__ TmaMap tmA, const __grid_constant__ TmaMap tmB";
    for (size_t i = 0; i < sdesc.size(); ++i) k << ", const __grid_constant__ TmaMap tmS" << i;
    k << ") {\n";
    k << "  typedef int idx_t;\n";
    k << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
    k << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
    k << "  unsigned long long* full = (unsigned long long*)(smem + " << REG << ");\n";
    k << "  unsigned long long* empty = full + " << S << ";\n";
    k << "  unsigned long long* accf = empty + " << S << ";\n";
    k << "  unsigned long long* sidef = accf + 1;\n  (void)sidef;\n";
    if (rasync) k << "  unsigned long long* rbar = accf + 2;\n  unsigned* tslot = (unsigned*)(accf + 3);\n";
    else k << "  unsigned* tslot = (unsigned*)(accf + 2);\n";
    k << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
    if (KS > 1)  // cluster of KS CTAs along x = the K-slices of one output tile
      k << "  const int ks = blockIdx.x % " << KS << ";\n  const int tile_m = (blockIdx.x / " << KS
        << ") * 128, tile_n = blockIdx.y * " << BN << ";\n";
    else k << "  const int ks = 0;\n  const int tile_m = blockIdx.x * 128, tile_n = blockIdx.y * " << BN << ";\n";
    k << "  int bzl = blockIdx.z;\n";
    k << "  const int bzlin = bzl;\n  (void)bzlin; (void)ks;\n";
    for (int b = nbC - 1; b >= 0; --b) {
      k << "  const int " << ep.batch_vars[b] << " = bzl % " << C[b] << "; bzl /= " << C[b] << ";\n";
    }
    k << "  (void)bzl;\n";
    // operand loads (variables kb, sa, sb, s in scope)
    std::ostringstream lda, ldb;
    if (a_kmaj) {
      lda << "      " << load(da.rank) << "(sa, &tmA, full + s, " << coords("kb * 64", "tile_m", ba_axes, va, true) << ");\n";
    } else {
      for (int cc = 0; cc < 2; ++cc)
        lda << "      " << load(da.rank) << "(sa + " << cc * 8192 << ", &tmA, full + s, "
            << coords("tile_m + " + str(cc * 64), "kb * 64", ba_axes, va, false) << ");\n";
    }
    if (b_kmaj) {
      ldb << "      " << load(db.rank) << "(sb, &tmB, full + s, " << coords("kb * 64", "tile_n", bb_axes, vb, true) << ");\n";
    } else {
      for (int cc = 0; cc < (BN + 63) / 64; ++cc)
        ldb << "      " << load(db.rank) << "(sb + " << cc * 8192 << ", &tmB, full + s, "
            << coords("tile_n + " + str(cc * 64), "kb * 64", bb_axes, vb, false) << ");\n";
    }
    // Operands that are graph inputs (weights) are never written by any kernel of a plan,
    // so their first PRE stages are fetched right after barrier init, before the
    // programmatic-dependency wait: under PDL the weight stream of this GEMM overlaps
    // the tail of the previous kernel.
    const bool earlyA = va.src.is_input, earlyB = vb.src.is_input;
    const int64_t PRE = (earlyA || earlyB) ? std::min<int64_t>(S, NK) : 0;
    // side tiles: one barrier for all of them; graph inputs load before the PDL wait
    auto side_load = [&](size_t i) {
      std::string c2 = "tile_n, tile_m";
      for (int b : sd_axes[i]) c2 += ", " + ep.batch_vars[b];
      return "    tma_load_" + std::to_string(sdesc[i].rank) + "d(smem + " + str(REG0 + side_off[i]) + ", &tmS" +
             std::to_string(i) + ", sidef, " + c2 + ");\n";
    };
    k << "  if (threadIdx.x == 0) {\n    for (int s = 0; s < " << S
      << "; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }\n"
      << "    mbar_init(accf, 1);\n    mbar_init(sidef, 1);\n" << (rasync ? "    mbar_init(rbar, 1);\n" : "")
      << "    mbar_fence_init();\n    tma_prefetch(&tmA);\n"
      << "    tma_prefetch(&tmB);\n";
    if (rasync) k << "    mbar_expect_tx(rbar, " << (int64_t)(KS - 1) * RO * BN * 4 << "u);\n";
    if (!sdesc.empty()) {
      int64_t tot = 0;
      for (auto& d : sdesc) tot += (int64_t)d.box[0] * d.box[1] * (d.dtype ? 2 : 4);
      k << "    mbar_expect_tx(sidef, " << tot << "u);\n";
      for (size_t i = 0; i < sdesc.size(); ++i)
        if (ep.ext[ep.sides[i].slot].is_input) k << side_load(i);
    }
    if (PRE) {
      k << "    for (int s = 0; s < " << PRE << "; ++s) {\n      const int kb = ks * " << NK << " + s;\n";
      k << "      mbar_expect_tx(full + s, " << STAGE << "u);\n";
      k << "      unsigned char* sa = smem + s * " << STAGE << ";\n      unsigned char* sb = sa + " << A_BYTES << ";\n";
      k << "      (void)sa; (void)sb; (void)kb;\n";
      if (earlyA) k << lda.str();
      if (earlyB) k << ldb.str();
      k << "    }\n";
    }
    k << "  }\n";
    k << "  if (warp == 2) tc_alloc(tslot, " << tcols << ");\n";
    k << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
    k << "  const unsigned tmem = *tslot;\n";
    // the receive barriers of every CTA of the cluster are armed before any push
    // (relaxed arrive: only the mbarrier inits, fenced by fence.mbarrier_init, must be seen)
    if (rasync) k << "  asm volatile(\"barrier.cluster.arrive.relaxed.aligned;\\nbarrier.cluster.wait.aligned;\" ::: \"memory\");\n";
    // Graph-input operands the epilogue reads with plain loads after the main loop (bias,
    // residual; never written inside a plan) are pulled into L2 before the dependency
    // wait, spread over the grid's threads: in a cold step their first touch is then an
    // L2 hit instead of an HBM round trip at the end of the critical path.
    {
      std::ostringstream pf;
      for (size_t i = 0; i < ep.ext.size(); ++i) {
        const Ref& r = ep.ext[i];
        if (!r.is_input || (r.id == va.src.id && va.src.is_input) || (r.id == vb.src.id && vb.src.is_input)) continue;
        bool staged = false;
        for (auto& sd : ep.sides) staged = staged || sd.slot == (int)i;
        const int64_t lines = (numel(g.shape_of(r)) * dtype_size(g.dtype_of(r)) + 127) / 128;
        if (staged || lines > (4 << 20) / 128) continue;
        pf << "    for (unsigned l = pf0; l < " << lines << "u; l += pfn)\n"
           << "      asm volatile(\"prefetch.global.L2 [%0];\" ::\"l\"((const char*)p" << i << " + (unsigned long long)l * 128));\n";
      }
      if (!pf.str().empty())
        k << "  {\n    const unsigned pfn = gridDim.x * gridDim.y * gridDim.z * blockDim.x;\n"
          << "    const unsigned pf0 = ((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * blockDim.x + threadIdx.x;\n"
          << pf.str() << "  }\n";
    }
    k << "  pdl_trigger();\n  pdl_wait();\n";
    // producer
    k << "  if (warp == 0 && lane == 0) {\n";
    for (size_t i = 0; i < sdesc.size(); ++i)
      if (!ep.ext[ep.sides[i].slot].is_input) k << side_load(i);
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = ks * " << NK << "; kb < (ks + 1) * " << NK << "; ++kb) {\n";
    k << "      const bool pre = kb - ks * " << NK << " < " << PRE << ";\n      (void)pre;\n";
    k << "      mbar_wait(empty + s, ph ^ 1u);\n";
    k << "      if (!pre) mbar_expect_tx(full + s, " << STAGE << "u);\n";
    k << "      unsigned char* sa = smem + s * " << STAGE << ";\n";
    k << "      unsigned char* sb = sa + " << A_BYTES << ";\n";
    k << (earlyA ? "      if (!pre) {\n" + lda.str() + "      }\n" : lda.str());
    k << (earlyB ? "      if (!pre) {\n" + ldb.str() + "      }\n" : ldb.str());
    k << "      if (++s == " << S << ") { s = 0; ph ^= 1u; }\n    }\n";
    // MMA issuer
    k << "  } else if (warp == 1 && lane == 0) {\n";
    k << "    int s = 0; unsigned ph = 0;\n";
    k << "    for (int kb = 0; kb < " << NK << "; ++kb) {\n";
    k << "      mbar_wait(full + s, ph);\n      tc_fence_after();\n";
    k << "      const unsigned sa = smem_u32(smem + s * " << STAGE << "), sb = sa + " << A_BYTES << ";\n";
    k << "      #pragma unroll\n      for (int k = 0; k < 4; ++k) {\n";
    k << "        const unsigned long long ad = umma_desc(sa + " << (a_kmaj ? "k * 32" : "k * 2048") << ", "
      << (a_kmaj ? 16 : 8192) << ", 1024);\n";
    if (b_kmaj)
      k << "        const unsigned long long bd = umma_desc(sb + k * 32, 16, 1024);\n";
    else
      k << "        const unsigned long long bd = umma_desc(sb + k * " << 16 * b_row_bytes << ", 8192, "
        << 8 * b_row_bytes << ", " << b_swz_umma << ");\n";
    k << "        tc_mma(tmem, ad, bd, " << idesc << "u, (kb | k) != 0);\n      }\n";
    k << "      tc_commit(empty + s);\n";
    k << "      if (++s == " << S << ") { s = 0; ph ^= 1u; }\n    }\n";
    k << "    tc_commit(accf);\n  }\n";
    // epilogue
    k << "  __syncwarp();\n  mbar_wait(accf, 0);\n  __syncwarp();\n  tc_fence_after();\n";
    if (KS == 1) {
      if (!sdesc.empty()) {
        for (size_t i = 0; i < sdesc.size(); ++i)
          k << "  const unsigned sside" << i << " = smem_u32(smem + " << REG0 + side_off[i] << ");\n";
        k << "  mbar_wait(sidef, 0);\n";
      }
      k << emit_tmem_epilogue(ep, BN, CW, TE, M, N);
    } else {
      if (rasync) k << emit_dsmem_splitk_async(ep, BN, CW, KS, M, N, "(smem + " + str(RECV_OFF) + ")", "rbar");
      else k << emit_dsmem_splitk(ep, BN, CW, KS, M, N, "true", "warp", 128);
    }
    k << "  tc_fence_before();\n  __syncthreads();\n";
    k << "  if (warp == 2) tc_dealloc(tmem, " << tcols << ");\n}\n";

    KernelVariant kv;
    std::string src = k.str();
    char nm[64];
    std::snprintf(nm, sizeof nm, "korch_gemm_%016llx",
                  (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + src));
    kv.name = nm;
    size_t pos = src.find("KNAME");
    src.replace(pos, 5, kv.name);
    kv.source = src;
    kv.tcgen05 = true;
    kv.block = 128;
    kv.grid = Mt * KS;
    kv.grid_y = Nt;
    kv.grid_z = batch;
    kv.cluster = KS;
    kv.smem = smem;
    da.tensor = slotA;
    db.tensor = slotB;
    kv.tma = {da, db};
    for (auto& d : sdesc) kv.tma.push_back(d);
    std::ostringstream t;
    t << "gemm BM=128 BN=" << BN << " BK=64 splitK=" << KS << " stages=" << S << " A=" << (a_kmaj ? "K" : "M")
      << "-major B=" << (b_kmaj ? "K" : "N") << "-major M=" << M << " N=" << N << " K=" << K << " batch=" << batch
      << (TE > 1 ? " epi=cl" : "") << (sdesc.empty() ? "" : " side=tma") << (rasync ? " red=st.async" : "");
    kv.tag = t.str();
    kp.variants.push_back(kv);
  }
  if (kp.variants.empty()) {
    if (gather_fallback) {
      KernelPlan gp = generate_matmul_gather(g, c, mm, va, vb);
      if (gp.klass != KORCH_CLASS_REJECTED) return gp;
      kp.reject += "; " + gp.reject;
    }
    return kp;
  }
  kp.klass = KORCH_CLASS_GEMM;
  kp.reject.clear();
  return kp;
}


// N2: fused two-GEMM attention candidate.  S = A1 * B1 lands
// in TMEM; the softmax-like chain from S to P (elementwise ops + in-tile row reductions,
// one thread per row) runs in registers and writes P as bf16 straight into shared memory
// in the canonical K-major 128B-swizzled layout; O = P * V is issued on the tensor core
// from that smem; O's fused epilogue (views folded into the store) writes the output.
// Q, K^T and V reach shared memory by TMA through their strided views.  P never
// touches HBM.  Single pass: the whole row (N1 <= 256) is in one tile.
KernelPlan generate_attention(const Graph& g, const Candidate& c) {
  KernelPlan kp;
  kp.klass = KORCH_CLASS_REJECTED;
  std::vector<int> lin;
  for (int m : c.members)
    if (g.is_dense_linear(m)) lin.push_back(m);
  if (lin.size() != 2) { kp.reject = "expected two linear primitives"; return kp; }
  if (g.topo_index[lin[0]] > g.topo_index[lin[1]]) std::swap(lin[0], lin[1]);
  const Prim& L1 = g.prims[lin[0]];
  const Prim& L2 = g.prims[lin[1]];
  if (L1.kind != Kind::MatMul || L2.kind != Kind::MatMul) { kp.reject = "attention needs two MatMuls"; return kp; }
  std::set<int> mem(c.members.begin(), c.members.end());
  if (L2.in[0].is_input || !mem.count(L2.in[0].id)) { kp.reject = "P must be computed in the kernel"; return kp; }
  const int pnode = L2.in[0].id;
  View vq, vk, vv;
  std::set<int> chain;
  std::string err;
  if (!operand_view(g, mem, L1, 0, &vq, &chain, &err) || !operand_view(g, mem, L1, 1, &vk, &chain, &err) ||
      !operand_view(g, mem, L2, 1, &vv, &chain, &err)) {
    kp.reject = err;
    return kp;
  }
  for (auto* v : {&vq, &vk, &vv})
    if (g.dtype_of(v->src) != DType::BF16 || (v->off * 2) % 16 || v->ksplit) {
      kp.reject = "attention operands must be aligned, unsplit bf16 views";
      return kp;
    }
  const Shape& SS = L1.shape;  // [batch..., M, N1]
  const Shape& OS = L2.shape;  // [batch..., M, N2]
  int nb = (int)SS.size() - 2;
  int64_t M = SS[nb], N1 = SS[nb + 1], K1 = vq.shape.back(), N2 = OS.back();
  if ((int)OS.size() != (int)SS.size() || (int)vq.shape.size() != nb + 2 || (int)vk.shape.size() != nb + 2 ||
      (int)vv.shape.size() != nb + 2) {
    kp.reject = "attention batch dims";
    return kp;
  }
  if (N1 % 64 || N1 > 256 || K1 > 128 || N2 % 16 || N2 > 256 || N1 + N2 > 512) {
    kp.reject = "attention tile limits (N1 % 64, N1 <= 256, K1 <= 128, N2 <= 256)";
    return kp;
  }
  bool q_k = vq.coef[nb + 1] == 1, k_k = vk.coef[nb] == 1, v_n = vv.coef[nb + 1] == 1, v_k = vv.coef[nb] == 1;
  if (!q_k || !k_k || !(v_n || v_k)) { kp.reject = "attention operand majorness"; return kp; }
  // pass 1: P from the S accumulator (full row, in-tile reductions)
  std::vector<Ref> pre{vq.src, vk.src, vv.src};
  GemmEpilogue ep1, ep2;
  if (!make_gemm_epilogue(g, c, lin[0], (int)N1, pre, &ep1, &err, pnode)) { kp.reject = "P: " + err; return kp; }
  if (!make_gemm_epilogue(g, c, lin[1], 32, ep1.ext, &ep2, &err)) { kp.reject = "O: " + err; return kp; }
  // column-lane O epilogue unless O is stored row-contiguous
  int TE2 = 1;
  if (!ep2.rows_unit) {
    GemmEpilogue e2;
    std::string e;
    if (make_gemm_epilogue(g, c, lin[1], 32, ep1.ext, &e2, &e, -1, 4) && e2.ext.size() == ep2.ext.size()) {
      ep2 = e2;
      TE2 = 4;
    }
  }
  kp.ext = ep2.ext;
  auto slot_of = [&](const Ref& r) {
    for (size_t i = 0; i < kp.ext.size(); ++i)
      if (kp.ext[i].is_input == r.is_input && kp.ext[i].id == r.id) return (int)i;
    return -1;
  };
  int sq = slot_of(vq.src), sk = slot_of(vk.src), sv = slot_of(vv.src);
  auto desc = [&](const View& v, int slot, int64_t inner, int64_t outer, int64_t outer_coef, uint32_t bi, uint32_t bo,
                  std::vector<int>* baxes, TmaDesc* d) {
    d->tensor = slot; d->dtype = 1; d->swizzle = 3; d->elem_off = v.off; d->rank = 0;
    auto push = [&](int64_t dim, int64_t st, uint32_t box) {
      d->dims[d->rank] = dim; d->strides[d->rank] = st * 2; d->box[d->rank] = box; d->rank++;
    };
    push(inner, 1, bi);
    push(outer, outer_coef ? outer_coef : inner, bo);
    for (int b = 0; b < nb; ++b)
      if (v.coef[b] != 0 && v.shape[b] > 1) {
        if (d->rank >= 5) return false;
        push(v.shape[b], v.coef[b], 1);
        baxes->push_back(b);
      }
    for (int i = 1; i < d->rank; ++i)
      if (d->strides[i] % 16) return false;
    return true;
  };
  TmaDesc dq, dk, dv;
  std::vector<int> bq, bk, bv;
  bool ok = desc(vq, sq, K1, M, vq.coef[nb], 64, 128, &bq, &dq) && desc(vk, sk, K1, N1, vk.coef[nb + 1], 64, (uint32_t)N1, &bk, &dk);
  ok = ok && (v_n ? desc(vv, sv, N2, N1, vv.coef[nb], 64, (uint32_t)N1, &bv, &dv)
                  : desc(vv, sv, N1, N2, vv.coef[nb + 1], 64, (uint32_t)N2, &bv, &dv));
  if (!ok) { kp.reject = "attention operand strides not expressible as TMA maps"; return kp; }
  int64_t batch = 1;
  for (int b = 0; b < nb; ++b) batch *= SS[b];
  const int64_t KB1 = (K1 + 63) / 64;
  const int Q_BYTES = (int)(KB1 * 16384), K_BYTES = (int)(KB1 * N1 * 128);
  const int V_BYTES = (int)(v_n ? ((N2 + 63) / 64) * N1 * 128 : (N1 / 64) * N2 * 128);
  const int P_BYTES = (int)((N1 / 64) * 16384);
  const int offK = Q_BYTES, offV = offK + K_BYTES, offP = offV + V_BYTES, offB = offP + P_BYTES;
  const int smem = offB + 64 + 1024;
  const int tcols = N1 + N2 <= 256 ? 256 : 512;
  const uint32_t id1 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N1 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t id2 = (1u << 4) | (1u << 7) | (1u << 10) | ((v_n ? 1u : 0u) << 16) | ((uint32_t)(N2 >> 3) << 17) |
                       ((uint32_t)(128 >> 4) << 24);
  kp.flops = 2.0 * batch * M * (N1 * K1 + N2 * N1);
  kp.bytes = ep2.bytes + ep1.bytes - 0 + 2 * (numel(vq.shape) + numel(vk.shape) + numel(vv.shape));
  auto coords = [&](const std::string& inner, const std::string& outer, const std::vector<int>& baxes) {
    std::string s = inner + ", " + outer;
    for (int b : baxes) s += ", " + std::string("bz") + std::to_string(b);
    return s;
  };
  auto load = [&](int rank) { return "tma_load_" + std::to_string(rank) + "d"; };
  // O epilogue: the column-lane mapping (TE2 = 4, staged through shared memory) and, as a
  // second launch variant, the row mapping (each thread stores its row's 64 contiguous
  // columns as 16-byte chunks: no staging round trip, L2 merges the row)
  std::vector<std::pair<GemmEpilogue, int>> ovars{{ep2, TE2}};
  if (TE2 > 1) {
    GemmEpilogue e1;
    std::string e;
    if (make_gemm_epilogue(g, c, lin[1], 32, ep1.ext, &e1, &e) && e1.ext.size() == ep2.ext.size()) ovars.push_back({e1, 1});
  }
  char nm[64];
  std::ostringstream t;
  t << "attention BM=128 N1=" << N1 << " K1=" << K1 << " N2=" << N2 << " V=" << (v_n ? "N" : "K") << "-major batch=" << batch;
  for (auto& ov : ovars) {
    const GemmEpilogue& ep2v = ov.first;
    const int TE2v = ov.second;
    std::ostringstream k;
    k << "extern \"C\" __global__ void __launch_bounds__(192, 1) KNAME(";
    for (size_t i = 0; i < kp.ext.size(); ++i)
      k << "const " << (g.dtype_of(kp.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
    k << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c) << ", "
      << "const __grid_constant__ TmaMap tmQ, const __grid_constant__ TmaMap tmK, const __grid_constant__ TmaMap tmV) {\n";
    k << "  typedef int idx_t;\n";
    k << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
    k << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
    k << "  unsigned long long* bars = (unsigned long long*)(smem + " << offB << ");\n";
    k << "  unsigned long long *ldf = bars, *sfull = bars + 1, *pfull = bars + 2, *ofull = bars + 3, *ldv = bars + 4;\n";
    k << "  unsigned* tslot = (unsigned*)(bars + 5);\n";
    k << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
    k << "  const int tile_m = blockIdx.x * 128;\n";
    k << "  int bzl = blockIdx.z;\n";
    for (int b = nb - 1; b >= 0; --b) k << "  const int bz" << b << " = bzl % " << SS[b] << "; bzl /= " << SS[b] << ";\n";
    k << "  (void)bzl;\n";
    k << "  if (threadIdx.x == 0) {\n    mbar_init(ldf, 1); mbar_init(sfull, 1); mbar_init(pfull, 4); mbar_init(ofull, 1);\n"
      << "    mbar_init(ldv, 1);\n"
      << "    mbar_fence_init();\n    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);\n  }\n";
    k << "  if (warp == 5) tc_alloc(tslot, " << tcols << ");\n";
    k << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
    k << "  const unsigned tmem = *tslot;\n";
    k << "  pdl_trigger();\n  pdl_wait();\n";
    // TMA: warp 4
    k << "  if (warp == 4 && lane == 0) {\n";
    // Q and K on one barrier, V on its own: S = QK^T and the softmax overlap V's arrival
    k << "    mbar_expect_tx(ldf, " << Q_BYTES + K_BYTES << "u);\n";
    k << "    mbar_expect_tx(ldv, " << V_BYTES << "u);\n";
    for (int64_t kb = 0; kb < KB1; ++kb) {
      k << "    " << load(dq.rank) << "(smem + " << kb * 16384 << ", &tmQ, ldf, " << coords(std::to_string(kb * 64), "tile_m", bq) << ");\n";
      k << "    " << load(dk.rank) << "(smem + " << offK + kb * N1 * 128 << ", &tmK, ldf, " << coords(std::to_string(kb * 64), "0", bk) << ");\n";
    }
    if (v_n) {
      for (int64_t cc = 0; cc < (N2 + 63) / 64; ++cc)
        k << "    " << load(dv.rank) << "(smem + " << offV + cc * N1 * 128 << ", &tmV, ldv, " << coords(std::to_string(cc * 64), "0", bv) << ");\n";
    } else {
      for (int64_t cc = 0; cc < N1 / 64; ++cc)
        k << "    " << load(dv.rank) << "(smem + " << offV + cc * N2 * 128 << ", &tmV, ldv, " << coords(std::to_string(cc * 64), "0", bv) << ");\n";
    }
    // MMA: warp 5
    k << "  } else if (warp == 5 && lane == 0) {\n";
    k << "    mbar_wait(ldf, 0);\n    tc_fence_after();\n";
    k << "    const unsigned sq = smem_u32(smem), sk = sq + " << offK << ", sv = sq + " << offV << ", sp = sq + " << offP << ";\n";
    k << "    #pragma unroll\n    for (int kb = 0; kb < " << KB1 << "; ++kb)\n";
    k << "      #pragma unroll\n      for (int k = 0; k < 4; ++k)\n";
    k << "        tc_mma(tmem, umma_desc(sq + kb * 16384 + k * 32, 16, 1024), umma_desc(sk + kb * " << N1 * 128
      << " + k * 32, 16, 1024), " << id1 << "u, (kb | k) != 0);\n";
    k << "    tc_commit(sfull);\n";
    k << "    mbar_wait(pfull, 0);\n    mbar_wait(ldv, 0);\n    tc_fence_after();\n";
    k << "    #pragma unroll\n    for (int k0 = 0; k0 < " << N1 << "; k0 += 16) {\n";
    k << "      const unsigned long long ad = umma_desc(sp + (k0 >> 6) * 16384 + (k0 & 63) * 2, 16, 1024);\n";
    if (v_n)
      k << "      const unsigned long long bd = umma_desc(sv + k0 * 128, " << N1 * 128 << ", 1024);\n";
    else
      k << "      const unsigned long long bd = umma_desc(sv + (k0 >> 6) * " << N2 * 128 << " + (k0 & 63) * 2, 16, 1024);\n";
    k << "      tc_mma(tmem + " << N1 << ", ad, bd, " << id2 << "u, k0 != 0);\n    }\n";
    k << "    tc_commit(ofull);\n  }\n";
    k << "  __syncwarp();\n";
    // epilogue warps 0-3: P into smem, then O to HBM
    k << "  if (warp < 4) {\n";
    k << "    const int gm = tile_m + warp * 32 + lane;\n    const int tid = 0;\n    (void)tid;\n";
    k << "    mbar_wait(sfull, 0);\n    __syncwarp();\n    tc_fence_after();\n";
    k << "    {\n      const int nb = 0;\n      float acc[" << N1 << "];\n";
    k << "      #pragma unroll\n      for (int q = 0; q < " << N1 / 32 << "; ++q)\n"
      << "        tc_ld32(tmem + ((unsigned)(warp * 32) << 16) + (unsigned)(q * 32), acc + q * 32);\n";
    k << ep1.body;
    k << "      const unsigned sp = smem_u32(smem + " << offP << ");\n";
    k << "      const int r = warp * 32 + lane;\n";
    k << "      #pragma unroll\n      for (int q = 0; q < " << N1 / 8 << "; ++q) {\n";
    k << "        uint4 pk = make_uint4(pack2(" << ep1.store << "[q * 8], " << ep1.store << "[q * 8 + 1]), pack2(" << ep1.store
      << "[q * 8 + 2], " << ep1.store << "[q * 8 + 3]), pack2(" << ep1.store << "[q * 8 + 4], " << ep1.store << "[q * 8 + 5]), pack2("
      << ep1.store << "[q * 8 + 6], " << ep1.store << "[q * 8 + 7]));\n";
    k << "        st_shared_v4(sp + (q >> 3) * 16384 + r * 128 + (((q & 7) ^ (r & 7)) << 4), pk);\n      }\n";
    k << "    }\n";
    k << "    fence_async_smem();\n    tc_fence_before();\n    __syncwarp();\n    if (lane == 0) mbar_arrive(pfull);\n";
    k << "    mbar_wait(ofull, 0);\n    __syncwarp();\n    tc_fence_after();\n";
    // O epilogue: Q/K/V/P shared memory is idle now (both MMAs done) and serves as the
    // column-lane staging buffer
    k << "    const int tile_n = 0;\n    const unsigned tmem_o = tmem + " << N1 << ";\n";
    k << "  " << emit_tmem_epilogue(ep2v, (int)((N2 + 31) / 32 * 32), 32, TE2v, M, N2, "tmem_o");
    k << "  }\n";
    k << "  tc_fence_before();\n  __syncthreads();\n";
    k << "  if (warp == 5) tc_dealloc(tmem, " << tcols << ");\n}\n";
    KernelVariant kv;
    std::string src = k.str();
    std::snprintf(nm, sizeof nm, "korch_attn_%016llx", (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + src));
    kv.name = nm;
    src.replace(src.find("KNAME"), 5, kv.name);
    kv.source = src;
    kv.tcgen05 = true;
    kv.block = 192;
    kv.grid = (M + 127) / 128;
    kv.grid_y = 1;
    kv.grid_z = batch;
    kv.smem = smem;
    kv.tma = {dq, dk, dv};
    kv.tag = t.str() + (TE2v != TE2 ? " O-epi=row" : "");
    kp.variants.push_back(kv);
  }
  kp.klass = KORCH_CLASS_GEMM;
  kp.reject.clear();

  // Variant 2: the softmax of S spread over 16 warps (4 threads per row).  TMEM lane
  // quarter q is readable by warps q, q+4, q+8, q+12; each loads a quarter of S's columns
  // for its 32 rows into a per-quarter staging buffer (named barrier per quarter), then
  // re-reads 8 rows x 4 lanes per row, so every thread owns N1/4 columns of one row and
  // the row reductions are 2-step shuffles: 4x less serial work per thread than one row
  // per thread.  Warps 16 / 17 issue TMA / MMA; the O epilogue stays on warps 0-3.
  if (N1 <= 128) {
    GemmEpilogue ep1s;
    std::string e3;
    if (make_gemm_epilogue(g, c, lin[0], (int)N1, pre, &ep1s, &e3, pnode, 4) && ep1s.ext.size() == ep1.ext.size() &&
        std::equal(ep1s.ext.begin(), ep1s.ext.end(), ep1.ext.begin(),
                   [](const Ref& a, const Ref& b) { return a.is_input == b.is_input && a.id == b.id; })) {
      const int CQ = (int)N1 / 4, PIT = (int)N1 + 4;
      const int offS = offP + P_BYTES, S_BYTES = 4 * 32 * PIT * 4;
      const int offB2 = offS + S_BYTES;
      const int smem2 = offB2 + 64 + 1024;
      std::ostringstream q;
      q << "extern \"C\" __global__ void __launch_bounds__(576, 1) KNAME(";
      for (size_t i = 0; i < kp.ext.size(); ++i)
        q << "const " << (g.dtype_of(kp.ext[i]) == DType::F32 ? "float" : "bf16_t") << "* __restrict__ p" << i << ", ";
      q << (g.prims[c.output].dtype == DType::F32 ? "float" : "bf16_t") << "* __restrict__ out" << extra_out_params(g, c) << ", "
        << "const __grid_constant__ TmaMap tmQ, const __grid_constant__ TmaMap tmK, const __grid_constant__ TmaMap tmV) {\n";
      q << "  typedef int idx_t;\n";
      q << "  extern __shared__ __align__(1024) unsigned char smem_raw[];\n";
      q << "  unsigned char* smem = (unsigned char*)(((unsigned long long)smem_raw + 1023ull) & ~1023ull);\n";
      q << "  unsigned long long* bars = (unsigned long long*)(smem + " << offB2 << ");\n";
      q << "  unsigned long long *ldf = bars, *sfull = bars + 1, *pfull = bars + 2, *ofull = bars + 3, *ldv = bars + 4;\n";
      q << "  unsigned* tslot = (unsigned*)(bars + 5);\n";
      q << "  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;\n";
      q << "  const int tile_m = blockIdx.x * 128;\n";
      q << "  int bzl = blockIdx.z;\n";
      for (int b = nb - 1; b >= 0; --b) q << "  const int bz" << b << " = bzl % " << SS[b] << "; bzl /= " << SS[b] << ";\n";
      q << "  (void)bzl;\n";
      q << "  if (threadIdx.x == 0) {\n    mbar_init(ldf, 1); mbar_init(sfull, 1); mbar_init(pfull, 16); mbar_init(ofull, 1);\n"
        << "    mbar_init(ldv, 1);\n"
        << "    mbar_fence_init();\n    tma_prefetch(&tmQ); tma_prefetch(&tmK); tma_prefetch(&tmV);\n  }\n";
      q << "  if (warp == 17) tc_alloc(tslot, " << tcols << ");\n";
      q << "  tc_fence_before();\n  __syncthreads();\n  tc_fence_after();\n";
      q << "  const unsigned tmem = *tslot;\n";
      q << "  pdl_trigger();\n  pdl_wait();\n";
      q << "  if (warp == 16 && lane == 0) {\n";
      q << "    mbar_expect_tx(ldf, " << Q_BYTES + K_BYTES << "u);\n";
      q << "    mbar_expect_tx(ldv, " << V_BYTES << "u);\n";
      for (int64_t kb = 0; kb < KB1; ++kb) {
        q << "    " << load(dq.rank) << "(smem + " << kb * 16384 << ", &tmQ, ldf, " << coords(std::to_string(kb * 64), "tile_m", bq) << ");\n";
        q << "    " << load(dk.rank) << "(smem + " << offK + kb * N1 * 128 << ", &tmK, ldf, " << coords(std::to_string(kb * 64), "0", bk) << ");\n";
      }
      if (v_n) {
        for (int64_t cc = 0; cc < (N2 + 63) / 64; ++cc)
          q << "    " << load(dv.rank) << "(smem + " << offV + cc * N1 * 128 << ", &tmV, ldv, " << coords(std::to_string(cc * 64), "0", bv) << ");\n";
      } else {
        for (int64_t cc = 0; cc < N1 / 64; ++cc)
          q << "    " << load(dv.rank) << "(smem + " << offV + cc * N2 * 128 << ", &tmV, ldv, " << coords(std::to_string(cc * 64), "0", bv) << ");\n";
      }
      q << "  } else if (warp == 17 && lane == 0) {\n";
      q << "    mbar_wait(ldf, 0);\n    tc_fence_after();\n";
      q << "    const unsigned sq = smem_u32(smem), sk = sq + " << offK << ", sv = sq + " << offV << ", sp = sq + " << offP << ";\n";
      q << "    #pragma unroll\n    for (int kb = 0; kb < " << KB1 << "; ++kb)\n";
      q << "      #pragma unroll\n      for (int k = 0; k < 4; ++k)\n";
      q << "        tc_mma(tmem, umma_desc(sq + kb * 16384 + k * 32, 16, 1024), umma_desc(sk + kb * " << N1 * 128
        << " + k * 32, 16, 1024), " << id1 << "u, (kb | k) != 0);\n";
      q << "    tc_commit(sfull);\n";
      q << "    mbar_wait(pfull, 0);\n    mbar_wait(ldv, 0);\n    tc_fence_after();\n";
      q << "    #pragma unroll\n    for (int k0 = 0; k0 < " << N1 << "; k0 += 16) {\n";
      q << "      const unsigned long long ad = umma_desc(sp + (k0 >> 6) * 16384 + (k0 & 63) * 2, 16, 1024);\n";
      if (v_n)
        q << "      const unsigned long long bd = umma_desc(sv + k0 * 128, " << N1 * 128 << ", 1024);\n";
      else
        q << "      const unsigned long long bd = umma_desc(sv + (k0 >> 6) * " << N2 * 128 << " + (k0 & 63) * 2, 16, 1024);\n";
      q << "      tc_mma(tmem + " << N1 << ", ad, bd, " << id2 << "u, k0 != 0);\n    }\n";
      q << "    tc_commit(ofull);\n  }\n";
      q << "  __syncwarp();\n";
      q << "  if (warp < 16) {\n";
      q << "    const int qq = warp & 3, cq = warp >> 2;\n";
      q << "    float* stq = reinterpret_cast<float*>(smem + " << offS << ") + qq * " << 32 * PIT << ";\n";
      q << "    mbar_wait(sfull, 0);\n    __syncwarp();\n    tc_fence_after();\n";
      q << "    {\n      float accq[" << CQ << "];\n";
      if (CQ == 16) q << "      tc_ld16(tmem + ((unsigned)(qq * 32) << 16) + (unsigned)(cq * 16), accq);\n";
      else
        q << "      #pragma unroll\n      for (int u = 0; u < " << CQ / 32 << "; ++u)\n        tc_ld32(tmem + ((unsigned)(qq * 32) << 16) + (unsigned)(cq * "
          << CQ << " + u * 32), accq + u * 32);\n";
      q << "      #pragma unroll\n      for (int u = 0; u < " << CQ / 4 << "; ++u)\n"
        << "        *reinterpret_cast<float4*>(stq + lane * " << PIT << " + cq * " << CQ << " + 4 * u) = make_float4(accq[4 * u], "
           "accq[4 * u + 1], accq[4 * u + 2], accq[4 * u + 3]);\n    }\n";
      q << "    asm volatile(\"bar.sync %0, 128;\" :: \"r\"(1 + qq) : \"memory\");\n";
      q << "    {\n      const int rq = cq * 8 + (lane >> 2), tid = lane & 3;\n";
      q << "      const int gm = tile_m + qq * 32 + rq;\n      const int nb = 0;\n      const unsigned gmask = 0xffffffffu;\n"
        << "      (void)gmask;\n";
      q << "      float acc[" << N1 / 4 << "];\n";
      q << "      #pragma unroll\n      for (int k = 0; k < " << N1 / 32 << "; ++k) {\n";
      q << "        const float4 a0 = *reinterpret_cast<const float4*>(stq + rq * " << PIT << " + (tid + k * 4) * 8);\n";
      q << "        const float4 a1 = *reinterpret_cast<const float4*>(stq + rq * " << PIT << " + (tid + k * 4) * 8 + 4);\n";
      q << "        acc[k * 8] = a0.x; acc[k * 8 + 1] = a0.y; acc[k * 8 + 2] = a0.z; acc[k * 8 + 3] = a0.w;\n";
      q << "        acc[k * 8 + 4] = a1.x; acc[k * 8 + 5] = a1.y; acc[k * 8 + 6] = a1.z; acc[k * 8 + 7] = a1.w;\n      }\n";
      q << ep1s.body;
      q << "      const unsigned sp = smem_u32(smem + " << offP << ");\n";
      q << "      const int r = qq * 32 + rq;\n";
      q << "      #pragma unroll\n      for (int k = 0; k < " << N1 / 32 << "; ++k) {\n";
      q << "        const int col = (tid + k * 4) * 8;\n";
      q << "        uint4 pk = make_uint4(pack2(" << ep1s.store << "[k * 8], " << ep1s.store << "[k * 8 + 1]), pack2(" << ep1s.store
        << "[k * 8 + 2], " << ep1s.store << "[k * 8 + 3]), pack2(" << ep1s.store << "[k * 8 + 4], " << ep1s.store
        << "[k * 8 + 5]), pack2(" << ep1s.store << "[k * 8 + 6], " << ep1s.store << "[k * 8 + 7]));\n";
      q << "        st_shared_v4(sp + (col >> 6) * 16384 + r * 128 + ((((col & 63) >> 3) ^ (r & 7)) << 4), pk);\n      }\n";
      q << "    }\n";
      q << "    fence_async_smem();\n    tc_fence_before();\n    __syncwarp();\n    if (lane == 0) mbar_arrive(pfull);\n";
      q << "    if (warp < 4) {\n";
      q << "      mbar_wait(ofull, 0);\n      __syncwarp();\n      tc_fence_after();\n";
      q << "      const int tile_n = 0;\n      const unsigned tmem_o = tmem + " << N1 << ";\n";
      q << "    " << emit_tmem_epilogue(ep2, (int)((N2 + 31) / 32 * 32), 32, TE2, M, N2, "tmem_o");
      q << "    }\n  }\n";
      q << "  tc_fence_before();\n  __syncthreads();\n";
      q << "  if (warp == 17) tc_dealloc(tmem, " << tcols << ");\n}\n";
      KernelVariant k2;
      std::string s2 = q.str();
      std::snprintf(nm, sizeof nm, "korch_attn_%016llx", (unsigned long long)fnv1a(std::string(kSm100GemmTemplate) + "\n" + s2));
      k2.name = nm;
      s2.replace(s2.find("KNAME"), 5, k2.name);
      k2.source = s2;
      k2.tcgen05 = true;
      k2.block = 576;
      k2.grid = (M + 127) / 128;
      k2.grid_y = 1;
      k2.grid_z = batch;
      k2.smem = smem2;
      k2.tma = {dq, dk, dv};
      k2.tag = t.str() + " softmax=4/row";
      if (smem2 <= 227 * 1024) kp.variants.push_back(k2);
    } else if (getenv("KORCH_GEN_TRACE")) {
      std::fprintf(stderr, "[attention split softmax] rejected: %s\n", e3.c_str());
    }
  }
  return kp;
}

}  // namespace korch
