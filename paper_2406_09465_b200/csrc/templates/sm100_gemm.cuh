// sm_100a building blocks for the KB5 GEMM template (tcgen05 + TMEM + TMA + mbarrier).
// Included (textually) ahead of every generated GEMM candidate kernel; NVRTC compiles
// the result for -arch=sm_100a.  No CUDA headers: everything is inline PTX.
//
// Roles inside one 128-thread CTA (one 128 x BN output tile per CTA):
//   warp 0 lane 0 : TMA producer   (cp.async.bulk.tensor -> smem ring, mbarrier full/empty)
//   warp 1 lane 0 : MMA issuer     (tcgen05.mma.cta_group::1.kind::f16, fp32 accum in TMEM)
//   warp 2        : TMEM allocator (tcgen05.alloc / dealloc)
//   warps 0-3     : epilogue       (tcgen05.ld 32x32b.x32 -> registers -> fused epilogue -> HBM)
#pragma once

struct __align__(64) TmaMap { unsigned long long v[16]; };

static __device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// ---------------------------------------------------------------- mbarrier
static __device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
static __device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// generic-proxy smem writes -> visible to the tensor core (async proxy)
static __device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
static __device__ __forceinline__ void st_shared_v4(unsigned addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
// 8 bf16 from shared memory (one 16-byte swizzle chunk) -> 8 floats
static __device__ __forceinline__ void ld_shared_bf16x8(unsigned addr, float* v) {
  unsigned a, b, c, d;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr) : "memory");
  v[0] = __uint_as_float(a << 16); v[1] = __uint_as_float(a & 0xffff0000u);
  v[2] = __uint_as_float(b << 16); v[3] = __uint_as_float(b & 0xffff0000u);
  v[4] = __uint_as_float(c << 16); v[5] = __uint_as_float(c & 0xffff0000u);
  v[6] = __uint_as_float(d << 16); v[7] = __uint_as_float(d & 0xffff0000u);
}
// 8 floats from shared memory (two 16-byte loads)
static __device__ __forceinline__ void ld_shared_f32x8(unsigned addr, float* v) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(addr) : "memory");
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]) : "r"(addr + 16u) : "memory");
}
static __device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

// ---------------------------------------------------------------- TMA
static __device__ __forceinline__ void tma_prefetch(const TmaMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((unsigned long long)m) : "memory");
}
static __device__ __forceinline__ void tma_load_2d(void* dst, const TmaMap* m, unsigned long long* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((unsigned long long)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
static __device__ __forceinline__ void tma_load_3d(void* dst, const TmaMap* m, unsigned long long* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((unsigned long long)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
static __device__ __forceinline__ void tma_load_4d(void* dst, const TmaMap* m, unsigned long long* bar, int c0, int c1, int c2,
                                                   int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((unsigned long long)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
static __device__ __forceinline__ void tma_load_5d(void* dst, const TmaMap* m, unsigned long long* bar, int c0, int c1, int c2,
                                                   int c3, int c4) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((unsigned long long)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05
// Shared-memory matrix descriptor (Blackwell version bits = 1).  layout: 2 = SWIZZLE_128B,
// 4 = SWIZZLE_64B, 6 = SWIZZLE_32B (bits 61-63).
static __device__ __forceinline__ unsigned long long umma_desc(unsigned saddr, unsigned lbo, unsigned sbo,
                                                               unsigned layout = 2) {
  unsigned long long d = 0;
  d |= (unsigned long long)((saddr >> 4) & 0x3FFF);
  d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;                  // version = 1 (sm_100)
  d |= (unsigned long long)layout << 61;
  return d;
}
static __device__ __forceinline__ void tc_alloc(unsigned* dst_smem, unsigned ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
static __device__ __forceinline__ void tc_dealloc(unsigned taddr, unsigned ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
static __device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_mma(unsigned tmem_d, unsigned long long adesc, unsigned long long bdesc, unsigned idesc,
                                              unsigned accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
static __device__ __forceinline__ void tc_commit(unsigned long long* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 32 lanes x 32 columns of fp32: thread i of the warp gets row (quarter*32 + i), 32 columns.
static __device__ __forceinline__ void tc_ld32(unsigned taddr, float* v) {
  unsigned r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 32 lanes x 16 columns (BN = 16 tiles).
static __device__ __forceinline__ void tc_ld16(unsigned taddr, float* v) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
static __device__ __forceinline__ bool elect_one() {
  unsigned pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

// 8 consecutive bf16 at a 2-byte-aligned global address: two aligned 16-byte read-only
// loads and a funnel shift (the second load only when the window straddles 16 bytes;
// it stays inside the 16-byte block holding the last requested element)
static __device__ __forceinline__ uint4 ld_bf16x8_unaligned(const unsigned short* p) {
  const unsigned long long a = (unsigned long long)p;
  const uint4* q = reinterpret_cast<const uint4*>(a & ~15ull);
  const unsigned off = (unsigned)(a & 15ull);
  const uint4 lo = __ldg(q);
  if (off == 0) return lo;
  const uint4 hi = __ldg(q + 1);
  const unsigned sh = (off & 3u) * 8u;
  unsigned w0, w1, w2, w3, w4;
  switch (off >> 2) {
    case 0: w0 = lo.x; w1 = lo.y; w2 = lo.z; w3 = lo.w; w4 = hi.x; break;
    case 1: w0 = lo.y; w1 = lo.z; w2 = lo.w; w3 = hi.x; w4 = hi.y; break;
    case 2: w0 = lo.z; w1 = lo.w; w2 = hi.x; w3 = hi.y; w4 = hi.z; break;
    default: w0 = lo.w; w1 = hi.x; w2 = hi.y; w3 = hi.z; w4 = hi.w; break;
  }
  uint4 r;
  r.x = __funnelshift_r(w0, w1, sh);
  r.y = __funnelshift_r(w1, w2, sh);
  r.z = __funnelshift_r(w2, w3, sh);
  r.w = __funnelshift_r(w3, w4, sh);
  return r;
}

// shared-memory reads for operands built from a staged tile (the conv halo)
static __device__ __forceinline__ uint4 ld_shared_v4(unsigned addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
static __device__ __forceinline__ unsigned short ld_shared_u16(unsigned addr) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
  return v;
}
// 8 consecutive bf16 at a 2-byte-aligned shared address (two aligned 16-byte reads and
// a funnel shift; the buffer keeps 16 readable bytes past its last element)
static __device__ __forceinline__ uint4 ld_shared_bf16x8_unaligned(unsigned addr) {
  const unsigned off = addr & 15u;
  const uint4 lo = ld_shared_v4(addr & ~15u);
  if (off == 0) return lo;
  const uint4 hi = ld_shared_v4((addr & ~15u) + 16u);
  const unsigned sh = (off & 3u) * 8u;
  unsigned w0, w1, w2, w3, w4;
  switch (off >> 2) {
    case 0: w0 = lo.x; w1 = lo.y; w2 = lo.z; w3 = lo.w; w4 = hi.x; break;
    case 1: w0 = lo.y; w1 = lo.z; w2 = lo.w; w3 = hi.x; w4 = hi.y; break;
    case 2: w0 = lo.z; w1 = lo.w; w2 = hi.x; w3 = hi.y; w4 = hi.z; break;
    default: w0 = lo.w; w1 = hi.x; w2 = hi.y; w3 = hi.z; w4 = hi.w; break;
  }
  uint4 r;
  r.x = __funnelshift_r(w0, w1, sh);
  r.y = __funnelshift_r(w1, w2, sh);
  r.z = __funnelshift_r(w2, w3, sh);
  r.w = __funnelshift_r(w3, w4, sh);
  return r;
}
// barrier over a subset of warps (id 1..15, n = thread count, a multiple of 32)
static __device__ __forceinline__ void named_bar_sync(unsigned id, unsigned n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---------------------------------------------------------------- clusters / DSMEM
// full cluster barrier (all threads of every CTA; release/acquire orders DSMEM traffic)
static __device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cta address in this CTA -> the same offset in CTA `rank` of the cluster
static __device__ __forceinline__ unsigned cluster_map(unsigned saddr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
static __device__ __forceinline__ void st_cluster_v4(unsigned caddr, float a, float b, float c, float d) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(caddr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}
