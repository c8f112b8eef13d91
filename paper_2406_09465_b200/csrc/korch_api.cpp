// C ABI (include/korch.h): graph load, enumeration, kernel generation/compilation,
// on-device profiling (PROFILING) and the executor.
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

#include <execinfo.h>
#include <signal.h>
#include <unistd.h>

#include "../../include/korch.h"
#include "codegen.h"
#include "cuda_api.h"
#include "enumerate.h"
#include "ir.h"

using namespace korch;

static thread_local std::string g_err = "no error";

static korch_status fail(korch_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define KORCH_TRY(...)                                             \
  try {                                                            \
    __VA_ARGS__                                                    \
  } catch (KorchError & e) {                                       \
    return fail(e.code, e.what());                                 \
  } catch (std::exception & e) {                                   \
    return fail(KORCH_E_ARG, std::string("internal: ") + e.what()); \
  }

#define CU_CHECK(expr)                                                        \
  do {                                                                        \
    CUresult _r = (expr);                                                     \
    if (_r != CUDA_SUCCESS) throw KorchError(KORCH_E_CUDA, std::string(#expr) + ": " + cu_err(_r)); \
  } while (0)

// ------------------------------------------------------------------ compiled kernels
struct Module {
  std::shared_ptr<const std::string> cubin;  // shared by the kernels of one NVRTC batch
  std::string log;
  bool compiled = false, failed = false;
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  CUdeviceptr scratch = 0;  // per-kernel scratch (split-K), zeroed once, kept zero by the kernel
  std::mutex mu;
};

struct korch_ctx {
  int device = -1;
  bool gpu = false;
  CUdevice dev = 0;
  CUcontext cuctx = nullptr;
  int sm_count = 0;
  int l2_bytes = 0;
  CUstream pstream = nullptr;           // profiling / capture stream
  std::vector<CUstream> aux;            // extra capture streams (concurrent plan branches, N4)
  std::vector<CUevent> events;          // capture-time fork / join / step-completion events
  CUdeviceptr arena = 0;
  size_t arena_bytes = 0;
  CUdeviceptr flush = 0;
  size_t flush_bytes = 0;
  std::mutex mu;
  std::mutex capture_mu;                // stream captures on pstream (execute, execute_host, profile)
  std::map<std::string, std::unique_ptr<Module>> modules;  // kernel name -> module
  std::map<const std::string*, CUmodule> loaded;           // batch cubin -> loaded module
  std::map<std::string, int64_t> timings;                  // kernel + protocol -> ns
  std::vector<std::shared_ptr<const std::string>> cubins;  // keeps loaded cubins alive

  void bind() {
    if (!gpu) throw KorchError(KORCH_E_CUDA, "host-only context (created with device -1)");
    CU_CHECK(cuda().cuCtxSetCurrent(cuctx));
  }
  Module* module_for(const std::string& name) {
    std::lock_guard<std::mutex> lk(mu);
    auto& m = modules[name];
    if (!m) m.reset(new Module());
    return m.get();
  }
  CUdeviceptr arena_get(size_t bytes) {
    if (bytes > arena_bytes) {
      if (arena) cuda().cuMemFree(arena);
      arena = 0;
      size_t b = std::max(bytes, (size_t)64 << 20);
      CUresult r = cuda().cuMemAlloc(&arena, b);
      if (r != CUDA_SUCCESS) throw KorchError(KORCH_E_OOM, "profiling arena: " + cu_err(r));
      arena_bytes = b;
    }
    return arena;
  }
};

struct CandState {
  bool planned = false;
  KernelPlan plan;
  int best = -1;          // chosen variant
  int64_t cost_ns = -1;
  std::vector<int64_t> var_ns;  // per-variant profiled time (-1 = not profiled)
  std::string sig;
};

struct BufRef {           // where a kernel argument lives at execute time
  enum { Input, Output, Work } kind = Input;
  int index = 0;          // input index / output index
  size_t offset = 0;      // workspace offset
};

struct Step {
  int cand = -1;
  int variant = 0;
  std::vector<BufRef> args;
  std::vector<BufRef> outs;  // the sink, then the secondary outputs (N1) in Candidate order
};

struct korch_graph {
  korch_ctx* ctx = nullptr;
  Graph g;
  bool enumerated = false;
  std::vector<Candidate> cands;
  std::vector<CandState> cs;
  int64_t n_states = 0;
  // accepted orchestration
  bool has_plan = false;
  std::vector<Step> steps;
  std::vector<std::vector<int>> deps;  // steps each step must follow (RAW / WAR / WAW on buffers)
  size_t ws_bytes = 0;
  // captured executable
  std::vector<const void*> cap_ptrs, cap_ptrs_host;
  CUgraphExec gexec = nullptr, gexec_host = nullptr;  // korch_execute / korch_execute_host
  std::mutex mu;
  ~korch_graph() {
    if (gexec && cuda().ok) cuda().cuGraphExecDestroy(gexec);
    if (gexec_host && cuda().ok) cuda().cuGraphExecDestroy(gexec_host);
  }
};

// ------------------------------------------------------------------ generation
static void ensure_planned(korch_graph* G, int64_t i) {
  CandState& s = G->cs[i];
  if (s.planned) return;
  s.plan = generate_kernel(G->g, G->cands[i]);
  Candidate& c = G->cands[i];
  c.klass = s.plan.klass;
  c.reject_reason = s.plan.reject;
  if (s.plan.klass != KORCH_CLASS_REJECTED) {
    c.bytes = s.plan.bytes;
    c.flops = s.plan.flops;
    c.signature = s.plan.variants[0].name;
  } else {
    c.signature = "rejected: " + s.plan.reject;
  }
  s.planned = true;
}

namespace korch {
extern const char* kSm100GemmTemplate;
}

static std::string full_source(const KernelVariant& v) {
  return kernel_prelude() + (v.tcgen05 ? std::string(kSm100GemmTemplate) + "\n" : std::string()) + v.source;
}

// NVRTC options of every kernel compile; part of the cache key
static const char* const kNvrtcOpts[] = {"-arch=sm_100a", "-std=c++17", "-default-device", "-lineinfo", "-DNDEBUG",
                                         "--diag-suppress=177,550"};

// Kernel names hash only the generated body (plus the GEMM template for tcgen05 kernels).
// Everything else that goes into the cubin -- the shared prelude, the template, the NVRTC
// options and the NVRTC version -- salts the cache key, so a change to any of them misses
// the on-disk cache instead of loading a stale cubin.
static const std::array<std::string, 2>& codegen_salt() {
  static const std::array<std::string, 2> salt = [] {
    std::string opts;
    for (const char* o : kNvrtcOpts) opts += std::string(o) + " ";
    int maj = 0, mnr = 0;
    if (nvrtc().ok && nvrtc().nvrtcVersion) nvrtc().nvrtcVersion(&maj, &mnr);
    opts += "nvrtc" + std::to_string(maj) + "." + std::to_string(mnr);
    char a[24], b[24];
    std::snprintf(a, sizeof a, "%016llx", (unsigned long long)fnv1a(kernel_prelude() + opts));
    std::snprintf(b, sizeof b, "%016llx",
                  (unsigned long long)fnv1a(kernel_prelude() + std::string(kSm100GemmTemplate) + opts));
    return std::array<std::string, 2>{a, b};
  }();
  return salt;
}

static std::string cache_key(const KernelVariant& v) { return v.name + "." + codegen_salt()[v.tcgen05 ? 1 : 0]; }

// Batched NVRTC compilation: up to kBatch kernels per program, so the per-program
// overhead (front-end start-up, prelude and template parsing) is paid once per batch.
// The batch cubin is shared by its kernels; the on-disk cache keeps one file per batch
// plus one small "<kernel>.ref" file per kernel naming it.
static constexpr size_t kBatch = 24;

static std::mutex g_cubin_mu;
static std::map<std::string, std::shared_ptr<const std::string>> g_cubin_files;  // path -> bytes

static std::shared_ptr<const std::string> read_file_cached(const std::string& path) {
  std::lock_guard<std::mutex> lk(g_cubin_mu);
  auto it = g_cubin_files.find(path);
  if (it != g_cubin_files.end()) return it->second;
  std::ifstream f(path, std::ios::binary);
  if (!f) return nullptr;
  std::stringstream ss;
  ss << f.rdbuf();
  auto p = std::make_shared<const std::string>(ss.str());
  if (p->empty()) return nullptr;
  g_cubin_files[path] = p;
  return p;
}

static void write_atomic(const std::string& path, const std::string& data);

// KORCH_CACHE_FALLBACK: a read-only older cache; kernels found there are copied into the
// current cache (batch cubin + ref), so rebuilding a cache keeps only live kernels
// without recompiling them
static bool cache_lookup(Module* m, const KernelVariant& v, const std::string& cache_dir) {
  if (cache_dir.empty()) return false;
  auto from = [&](const std::string& dir) -> std::shared_ptr<const std::string> {
    std::ifstream ref(dir + "/" + cache_key(v) + ".ref");
    if (!ref) return nullptr;
    std::string batch;
    std::getline(ref, batch);
    auto bytes = read_file_cached(dir + "/" + batch);
    if (bytes && dir != cache_dir) {
      std::ifstream have(cache_dir + "/" + batch);
      if (!have) write_atomic(cache_dir + "/" + batch, *bytes);
      write_atomic(cache_dir + "/" + cache_key(v) + ".ref", batch + "\n");
    }
    return bytes;
  };
  auto bytes = from(cache_dir);
  const char* fb = getenv("KORCH_CACHE_FALLBACK");
  if (!bytes && fb && *fb) bytes = from(fb);
  if (!bytes) return false;
  m->cubin = bytes;
  m->compiled = true;
  return true;
}

static bool nvrtc_compile(const std::string& src, const std::string& name, std::string* cubin, std::string* log) {
  NvrtcApi& nv = nvrtc();
  if (!nv.ok) {
    *log = nv.err;
    return false;
  }
  nvrtcProgram prog;
  if (nv.nvrtcCreateProgram(&prog, src.c_str(), (name + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    *log = "nvrtcCreateProgram failed";
    return false;
  }
  nvrtcResult r = nv.nvrtcCompileProgram(prog, (int)(sizeof kNvrtcOpts / sizeof kNvrtcOpts[0]),
                                         const_cast<const char**>(kNvrtcOpts));
  size_t ls = 0;
  nv.nvrtcGetProgramLogSize(prog, &ls);
  std::string lg(ls, '\0');
  if (ls) nv.nvrtcGetProgramLog(prog, &lg[0]);
  if (r != NVRTC_SUCCESS) {
    *log = std::string("NVRTC: ") + nv.nvrtcGetErrorString(r) + "\n" + lg;
    nv.nvrtcDestroyProgram(&prog);
    return false;
  }
  size_t cs = 0;
  nv.nvrtcGetCUBINSize(prog, &cs);
  cubin->resize(cs);
  nv.nvrtcGetCUBIN(prog, &(*cubin)[0]);
  nv.nvrtcDestroyProgram(&prog);
  return true;
}

static void write_atomic(const std::string& path, const std::string& data) {
  // unique per process and thread: several ranks may fill one cache directory at once
  std::string tmp = path + ".tmp" + std::to_string((long)getpid()) + "_" +
                    std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
  {
    std::ofstream f(tmp, std::ios::binary);
    f.write(data.data(), (std::streamsize)data.size());
  }
  std::rename(tmp.c_str(), path.c_str());
}

// Compile one batch of kernels into a single cubin; on failure retry them one by one
// so a bad kernel only rejects itself.
static void compile_batch(const std::vector<std::pair<Module*, const KernelVariant*>>& jobs, const std::string& cache_dir) {
  if (jobs.empty()) return;
  bool tc = false;
  std::string names;
  for (auto& j : jobs) {
    tc = tc || j.second->tcgen05;
    names += j.second->name + ";";
  }
  std::string src = kernel_prelude() + (tc ? std::string(kSm100GemmTemplate) + "\n" : std::string());
  for (auto& j : jobs) src += j.second->source + "\n";
  char bname[64];
  std::snprintf(bname, sizeof bname, "batch_%016llx.cubin", (unsigned long long)fnv1a(names + src));
  std::string cubin, log;
  if (nvrtc_compile(src, bname, &cubin, &log)) {
    auto shared = std::make_shared<const std::string>(std::move(cubin));
    if (!cache_dir.empty()) {
      write_atomic(cache_dir + "/" + bname, *shared);
      for (auto& j : jobs) write_atomic(cache_dir + "/" + cache_key(*j.second) + ".ref", std::string(bname) + "\n");
    }
    for (auto& j : jobs) {
      std::lock_guard<std::mutex> lk(j.first->mu);
      j.first->cubin = shared;
      j.first->compiled = true;
    }
    return;
  }
  if (jobs.size() == 1) {
    std::lock_guard<std::mutex> lk(jobs[0].first->mu);
    jobs[0].first->failed = true;
    jobs[0].first->log = log;
    return;
  }
  for (auto& j : jobs) compile_batch({j}, cache_dir);
}

static void compile_many(korch_graph* G, const std::vector<int64_t>& idx, int threads, const std::string& cache_dir) {
  std::vector<std::pair<Module*, const KernelVariant*>> jobs;
  std::map<Module*, bool> seen;
  for (int64_t i : idx) {
    ensure_planned(G, i);
    CandState& s = G->cs[i];
    if (s.plan.klass == KORCH_CLASS_REJECTED) continue;
    for (auto& v : s.plan.variants) {
      Module* m = G->ctx->module_for(v.name);
      {
        std::lock_guard<std::mutex> lk(m->mu);
        if (m->compiled || m->failed || seen.count(m)) continue;
        if (cache_lookup(m, v, cache_dir)) continue;
      }
      seen[m] = true;
      jobs.push_back({m, &v});
    }
  }
  // batches group kernels of one kind (tcgen05 kernels share the GEMM template)
  std::stable_sort(jobs.begin(), jobs.end(), [](const std::pair<Module*, const KernelVariant*>& a,
                                                const std::pair<Module*, const KernelVariant*>& b) {
    return a.second->tcgen05 < b.second->tcgen05;
  });
  std::vector<std::vector<std::pair<Module*, const KernelVariant*>>> batches;
  for (auto& j : jobs) {
    if (batches.empty() || batches.back().size() >= kBatch || batches.back().back().second->tcgen05 != j.second->tcgen05)
      batches.emplace_back();
    batches.back().push_back(j);
  }
  if (threads <= 0) {
    // NVRTC holds ~0.5-1 GB per in-flight tcgen05 batch: bound the parallelism
    const char* e = getenv("KORCH_COMPILE_THREADS");
    threads = e ? atoi(e) : (int)std::min(24u, std::max(1u, std::thread::hardware_concurrency()));
    if (threads <= 0) threads = 1;
  }
  threads = std::min<int>(threads, (int)std::max<size_t>(1, batches.size()));
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (;;) {
      size_t k = next++;
      if (k >= batches.size()) break;
      compile_batch(batches[k], cache_dir);
    }
  };
  std::vector<std::thread> ts;
  for (int t = 1; t < threads; ++t) ts.emplace_back(worker);
  worker();
  for (auto& t : ts) t.join();
}

static std::string default_cache_dir() {
  const char* e = getenv("KORCH_CACHE_DIR");
  return e ? e : "";
}

static CUfunction load_fn(korch_ctx* ctx, Module* m, const KernelVariant& v) {
  std::lock_guard<std::mutex> lk(m->mu);
  if (m->fn) return m->fn;
  if (!m->compiled) throw KorchError(KORCH_E_NVRTC, "kernel not compiled: " + m->log);
  {
    std::lock_guard<std::mutex> lk2(ctx->mu);
    auto it = ctx->loaded.find(m->cubin.get());
    if (it == ctx->loaded.end()) {
      CUmodule mod;
      CU_CHECK(cuda().cuModuleLoadData(&mod, m->cubin->data()));
      it = ctx->loaded.emplace(m->cubin.get(), mod).first;
      ctx->cubins.push_back(m->cubin);
    }
    m->mod = it->second;
  }
  CU_CHECK(cuda().cuModuleGetFunction(&m->fn, m->mod, v.name.c_str()));
  if (v.smem > 48 * 1024)
    CU_CHECK(cuda().cuFuncSetAttribute(m->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, v.smem));
  return m->fn;
}

// Load the kernel and allocate its scratch; must run outside stream capture.
static void prepare_variant(korch_ctx* ctx, const KernelVariant& v) {
  Module* m = ctx->module_for(v.name);
  load_fn(ctx, m, v);
  std::lock_guard<std::mutex> lk(m->mu);
  if (v.scratch_bytes > 0 && !m->scratch) {
    CUresult r = cuda().cuMemAlloc(&m->scratch, (size_t)v.scratch_bytes);
    if (r != CUDA_SUCCESS) throw KorchError(KORCH_E_OOM, "kernel scratch: " + cu_err(r));
    CU_CHECK(cuda().cuMemsetD8Async(m->scratch, 0, (size_t)v.scratch_bytes, nullptr));
    CU_CHECK(cuda().cuCtxSynchronize());
  }
}

// ------------------------------------------------------------------ launching
static void encode_tma(const TmaDesc& d, const void* base, CUtensorMap* out) {
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], es[5];
  int esz = d.dtype == 0 ? 4 : 2;
  for (int i = 0; i < d.rank; ++i) {
    dims[i] = (cuuint64_t)d.dims[i];
    box[i] = d.box[i];
    es[i] = 1;
    if (i > 0) strides[i - 1] = (cuuint64_t)d.strides[i];
  }
  const char* p = static_cast<const char*>(base) + d.elem_off * esz;
  CU_CHECK(cuda().cuTensorMapEncodeTiled(
      out, d.dtype == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, (cuuint32_t)d.rank,
      const_cast<char*>(p), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      (CUtensorMapSwizzle)d.swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
}

static void launch_variant(korch_ctx* ctx, const KernelPlan& plan, int vi, const std::vector<const void*>& ins,
                           const std::vector<void*>& outs, CUstream stream, bool pdl = false) {
  const KernelVariant& v = plan.variants[vi];
  Module* m = ctx->module_for(v.name);
  CUfunction fn = load_fn(ctx, m, v);
  if (outs.empty()) throw KorchError(KORCH_E_ARG, "kernel launched without an output buffer");
  void* out = outs[0];
  std::vector<CUdeviceptr> ptrs(ins.size() + outs.size());
  std::vector<void*> args;
  args.reserve(ins.size() + outs.size() + 1 + v.tma.size());
  for (size_t i = 0; i < ins.size(); ++i) {
    ptrs[i] = (CUdeviceptr)ins[i];
    args.push_back(&ptrs[i]);
  }
  for (size_t k = 0; k < outs.size(); ++k) {  // out, then the secondary outputs out1.. (N1)
    ptrs[ins.size() + k] = (CUdeviceptr)outs[k];
    args.push_back(&ptrs[ins.size() + k]);
  }
  CUdeviceptr scratch = m->scratch;
  if (v.scratch_bytes > 0) {
    if (!scratch) throw KorchError(KORCH_E_CUDA, "kernel scratch not prepared: " + v.name);
    args.push_back(&scratch);
  }
  std::vector<CUtensorMap> maps(v.tma.size());
  for (size_t t = 0; t < v.tma.size(); ++t) {
    const TmaDesc& d = v.tma[t];
    const void* base = d.tensor == -2 ? out : d.tensor == -3 ? (const void*)scratch : ins.at(d.tensor);
    encode_tma(d, base, &maps[t]);
    args.push_back(&maps[t]);
  }
  if (v.cluster > 1 || pdl) {
    CUlaunchConfig cfg{};
    cfg.gridDimX = (unsigned)v.grid;
    cfg.gridDimY = (unsigned)v.grid_y;
    cfg.gridDimZ = (unsigned)v.grid_z;
    cfg.blockDimX = (unsigned)v.block;
    cfg.blockDimY = cfg.blockDimZ = 1;
    cfg.sharedMemBytes = (unsigned)v.smem;
    cfg.hStream = stream;
    CUlaunchAttribute at[2];
    unsigned na = 0;
    if (v.cluster > 1) {
      at[na].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
      at[na].value.clusterDim.x = (unsigned)v.cluster;
      at[na].value.clusterDim.y = at[na].value.clusterDim.z = 1;
      ++na;
    }
    if (pdl) {  // programmatic dependent launch (the kernel calls griddepcontrol.wait)
      at[na].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
      at[na].value.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    CU_CHECK(cuda().cuLaunchKernelEx(&cfg, fn, args.data(), nullptr));
  } else {
    CU_CHECK(cuda().cuLaunchKernel(fn, (unsigned)v.grid, (unsigned)v.grid_y, (unsigned)v.grid_z, (unsigned)v.block, 1, 1, (unsigned)v.smem, stream,
                                   args.data(), nullptr));
  }
}

static int64_t tensor_bytes(const Graph& g, const Ref& r) { return numel(g.shape_of(r)) * dtype_size(g.dtype_of(r)); }

// Seeded synthetic operands for the profiler ("allocate seeded inputs
// at the candidate's exact shapes"): element i of a buffer with seed s is
// u = hash(s, i) / 2^32 mapped to [-1, 1), stored as f32 or bf16 (round to nearest even).
// A counter-based hash, so every buffer is reproducible and no host data is uploaded.
static const KernelVariant& fill_variant() {
  static KernelVariant v = [] {
    KernelVariant k;
    k.name = "korch_fill_v1";
    k.block = 256;
    k.source =
        "KI unsigned korch_hash(unsigned s, unsigned long long i) {\n"
        "  unsigned long long z = i * 0x9E3779B97F4A7C15ull + ((unsigned long long)s << 32) + s;\n"
        "  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull; z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;\n"
        "  return (unsigned)((z ^ (z >> 31)) >> 32);\n}\n"
        "KI float korch_u11(unsigned h) { return (float)(h >> 8) * (1.0f / 8388608.0f) - 1.0f; }\n"
        "extern \"C\" __global__ void __launch_bounds__(256) korch_fill_v1(unsigned* __restrict__ dst, "
        "unsigned long long nwords, unsigned seed, int bf16) {\n"
        "  for (unsigned long long w = blockIdx.x * 256ull + threadIdx.x; w < nwords; w += gridDim.x * 256ull) {\n"
        "    if (bf16) dst[w] = pack2(korch_u11(korch_hash(seed, 2 * w)), korch_u11(korch_hash(seed, 2 * w + 1)));\n"
        "    else dst[w] = __float_as_uint(korch_u11(korch_hash(seed, w)));\n"
        "  }\n}\n";
    return k;
  }();
  return v;
}

static void prepare_fill(korch_ctx* ctx) {
  const KernelVariant& v = fill_variant();
  Module* m = ctx->module_for(v.name);
  if (!m->compiled && !m->failed) compile_batch({{m, &v}}, default_cache_dir());
  if (!m->compiled) throw KorchError(KORCH_E_NVRTC, "profiler fill kernel: " + m->log);
  load_fn(ctx, m, v);
}

// fill `elems` elements of dtype `dt` at `p` (the buffer is 256-byte padded, so the last
// bf16 word may cover one padding element)
static void launch_fill(korch_ctx* ctx, CUdeviceptr p, size_t elems, DType dt, unsigned seed, CUstream stream) {
  Module* m = ctx->module_for(fill_variant().name);
  const int bf = dt == DType::BF16;
  unsigned long long nwords = bf ? (elems + 1) / 2 : elems;
  unsigned grid = (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(8 * 148, (nwords + 255) / 256));
  void* args[] = {&p, &nwords, &seed, (void*)&bf};
  CU_CHECK(cuda().cuLaunchKernel(m->fn, grid, 1, 1, 256, 1, 1, 0, stream, args, nullptr));
}

// Launch the plan's steps into the capture running on ctx->pstream.  With KORCH_STREAMS
// = k > 1 (default 4) independent steps go to different streams of the capture, so the
// graph has parallel branches (overlap-aware execution): a step joins
// the stream whose last step is one of its ancestors (the most recent one first, then a
// fresh stream, else the oldest), waits on events of the dependencies that stream order
// does not already imply, and keeps programmatic dependent launch behind the previous
// kernel of its stream (never for a stream's first plan kernel: graph inputs may still be
// in flight from host copies).  k = 1 is the sequential chain of reading A6.
template <typename LaunchFn>
static void capture_steps(korch_ctx* ctx, korch_graph* G, bool use_pdl, LaunchFn launch) {
  CudaApi& cu = cuda();
  const char* env = getenv("KORCH_STREAMS");  // read per capture (tests compare settings)
  const int ns = std::max(1, std::min(env ? atoi(env) : 4, 8));
  const size_t nsteps = G->steps.size();
  while ((int)ctx->aux.size() < ns - 1) {
    CUstream st;
    CU_CHECK(cu.cuStreamCreate(&st, CU_STREAM_NON_BLOCKING));
    ctx->aux.push_back(st);
  }
  while (ctx->events.size() < nsteps + 2 * (size_t)ns) {
    CUevent ev;
    CU_CHECK(cu.cuEventCreate(&ev, CU_EVENT_DISABLE_TIMING));
    ctx->events.push_back(ev);
  }
  std::vector<CUstream> streams{ctx->pstream};
  for (int i = 0; i + 1 < ns; ++i) streams.push_back(ctx->aux[i]);
  if (ns > 1) {  // fork: every aux stream joins the capture after what pstream has so far
    CUevent fork = ctx->events[nsteps];
    CU_CHECK(cu.cuEventRecord(fork, ctx->pstream));
    for (int i = 1; i < ns; ++i) CU_CHECK(cu.cuStreamWaitEvent(streams[i], fork, 0));
  }
  std::vector<int> last(ns, -1), where(nsteps, 0);
  std::vector<std::vector<char>> anc(nsteps, std::vector<char>(nsteps, 0));
  for (size_t t = 0; t < nsteps; ++t) {
    const std::vector<int>& D = G->deps[t];
    for (int d : D) {
      anc[t][d] = 1;
      for (size_t a = 0; a < nsteps; ++a) anc[t][a] = anc[t][a] || anc[d][a];
    }
    int sel = -1;
    if (ns == 1) sel = 0;
    else {
      int best = -2;
      for (int s = 0; s < ns; ++s) {  // the stream whose last step is the latest ancestor
        int L = last[s];
        if (L >= 0 && anc[t][L] && L > best) { best = L; sel = s; }
      }
      if (sel < 0)
        for (int s = 0; s < ns && sel < 0; ++s)
          if (last[s] < 0) sel = s;
      if (sel < 0) {
        int oldest = 1 << 30;
        for (int s = 0; s < ns; ++s)
          if (last[s] < oldest) { oldest = last[s]; sel = s; }
      }
    }
    const int L = last[sel];
    for (int d : D)
      if (where[d] != sel || d > L)  // not implied by this stream's order
        if (!(L >= 0 && (L == d || anc[L][d]))) CU_CHECK(cu.cuStreamWaitEvent(streams[sel], ctx->events[d], 0));
    launch(G->steps[t], streams[sel], use_pdl && L >= 0);
    if (ns > 1) CU_CHECK(cu.cuEventRecord(ctx->events[t], streams[sel]));
    last[sel] = (int)t;
    where[t] = sel;
  }
  for (int s = 1; s < ns; ++s) {  // join
    CUevent j = ctx->events[nsteps + ns + s];
    CU_CHECK(cu.cuEventRecord(j, streams[s]));
    CU_CHECK(cu.cuStreamWaitEvent(ctx->pstream, j, 0));
  }
}

// ------------------------------------------------------------------ API
extern "C" {

// the codegen salt identifies the prelude / template / NVRTC options the kernels are built
// with: profiled costs recorded under another version describe other kernels
const char* korch_version(void) {
  static const std::string v = "korch-b200 0.2 (sm_100a) codegen " + codegen_salt()[0] + "-" + codegen_salt()[1];
  return v.c_str();
}
const char* korch_last_error(void) { return g_err.c_str(); }

// KORCH_SEGV_TRACE=1: print a native backtrace on SIGSEGV (diagnostics on the GPU box,
// which has no debugger)
static void segv_trace(int sig) {
  void* fr[64];
  int n = backtrace(fr, 64);
  const char msg[] = "korch: fatal signal, native backtrace:\n";
  (void)!write(2, msg, sizeof msg - 1);
  backtrace_symbols_fd(fr, n, 2);
  signal(sig, SIG_DFL);
  raise(sig);
}

korch_status korch_create(int32_t device, korch_ctx** out) {
  if (!out) return fail(KORCH_E_ARG, "out is NULL");
  if (getenv("KORCH_SEGV_TRACE")) signal(SIGSEGV, segv_trace);
  KORCH_TRY({
    std::unique_ptr<korch_ctx> c(new korch_ctx());
    c->device = device;
    if (device >= 0) {
      CudaApi& cu = cuda();
      if (!cu.ok) return fail(KORCH_E_CUDA, cu.err);
      CU_CHECK(cu.cuDeviceGet(&c->dev, device));
      CU_CHECK(cu.cuDevicePrimaryCtxRetain(&c->cuctx, c->dev));
      CU_CHECK(cu.cuCtxSetCurrent(c->cuctx));
      CU_CHECK(cu.cuDeviceGetAttribute(&c->sm_count, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, c->dev));
      CU_CHECK(cu.cuDeviceGetAttribute(&c->l2_bytes, CU_DEVICE_ATTRIBUTE_L2_CACHE_SIZE, c->dev));
      CU_CHECK(cu.cuStreamCreate(&c->pstream, CU_STREAM_NON_BLOCKING));
      c->gpu = true;
    }
    *out = c.release();
    return KORCH_OK;
  })
}

korch_status korch_destroy(korch_ctx* c) {
  if (!c) return KORCH_OK;
  if (c->gpu && cuda().ok) {
    cuda().cuCtxSetCurrent(c->cuctx);
    cuda().cuCtxSynchronize();
    for (auto& kv : c->loaded) cuda().cuModuleUnload(kv.second);
    for (auto& kv : c->modules)
      if (kv.second->scratch) cuda().cuMemFree(kv.second->scratch);
    if (c->arena) cuda().cuMemFree(c->arena);
    if (c->flush) cuda().cuMemFree(c->flush);
    if (c->pstream) cuda().cuStreamDestroy(c->pstream);
    for (CUstream st : c->aux) cuda().cuStreamDestroy(st);
    for (CUevent ev : c->events) cuda().cuEventDestroy(ev);
    cuda().cuDevicePrimaryCtxRelease(c->dev);
  }
  delete c;
  return KORCH_OK;
}

korch_status korch_graph_load(korch_ctx* ctx, const char* json, size_t n, korch_graph** out) {
  if (!ctx || !json || !out) return fail(KORCH_E_ARG, "NULL argument");
  KORCH_TRY({
    std::unique_ptr<korch_graph> G(new korch_graph());
    G->ctx = ctx;
    G->g = load_graph(json, n);
    *out = G.release();
    return KORCH_OK;
  })
}

korch_status korch_graph_free(korch_graph* g) {
  if (g && g->ctx && g->ctx->gpu && cuda().ok) cuda().cuCtxSetCurrent(g->ctx->cuctx);
  delete g;
  return KORCH_OK;
}

korch_status korch_graph_info(const korch_graph* G, int32_t* np, int32_t* ni, int32_t* no) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (np) *np = (int32_t)G->g.prims.size();
  if (ni) *ni = (int32_t)G->g.inputs.size();
  if (no) *no = (int32_t)G->g.outputs.size();
  return KORCH_OK;
}

static korch_status write_buf(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (!buf || cap < s.size() + 1) return fail(KORCH_E_ARG, "buffer too small");
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return KORCH_OK;
}

korch_status korch_graph_dump(const korch_graph* G, char* buf, size_t cap, size_t* needed) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  KORCH_TRY({ return write_buf(dump_graph(G->g), buf, cap, needed); })
}

korch_status korch_validate(const korch_graph* G, char* report, size_t cap) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  KORCH_TRY({
    std::string r = validate_graph(G->g);
    size_t need;
    return write_buf(r, report, cap, &need);
  })
}

korch_status korch_enumerate(korch_graph* G, const korch_enum_opts* o, int64_t* n_cands, int64_t* n_states) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  KORCH_TRY({
    EnumOpts eo;
    if (o) {
      if (o->max_prims > 0) eo.max_prims = o->max_prims;
      eo.keep_multi_linear = o->keep_multi_linear != 0;
      if (o->max_states > 0) eo.max_states = o->max_states;
      if (o->partition_max > 0) eo.partition_max = o->partition_max;
      eo.attention_pairs = o->attention_pairs != 0;
      if (o->max_outputs > 1) eo.max_outputs = std::min<int32_t>(o->max_outputs, 4);
    }
    std::lock_guard<std::mutex> lk(G->mu);
    G->cands = enumerate_candidates(G->g, eo, &G->n_states);
    G->cs.assign(G->cands.size(), CandState());
    for (size_t i = 0; i < G->cands.size(); ++i) ensure_planned(G, (int64_t)i);
    G->enumerated = true;
    G->has_plan = false;
    if (n_cands) *n_cands = (int64_t)G->cands.size();
    if (n_states) *n_states = G->n_states;
    return KORCH_OK;
  })
}

korch_status korch_candidate(const korch_graph* G, int64_t i, korch_cand_desc* d) {
  if (!G || !d) return fail(KORCH_E_ARG, "NULL argument");
  if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
  const Candidate& c = G->cands[i];
  d->n_members = (int32_t)c.members.size();
  d->members = c.members.data();
  d->output = c.output;
  d->n_inputs = (int32_t)c.inputs.size();
  d->inputs = c.inputs.data();
  d->n_graph_inputs = (int32_t)c.graph_inputs.size();
  d->graph_inputs = c.graph_inputs.data();
  d->klass = c.klass;
  d->n_dense_linear = c.n_dense;
  d->bytes = c.bytes;
  d->flops = c.flops;
  d->signature = c.signature.c_str();
  d->part = c.part;
  d->n_extra_outputs = (int32_t)c.extra_outputs.size();
  d->extra_outputs = c.extra_outputs.data();
  return KORCH_OK;
}

korch_status korch_candidate_source(korch_graph* G, int64_t i, char* buf, size_t cap, size_t* needed) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
  KORCH_TRY({
    ensure_planned(G, i);
    const CandState& s = G->cs[i];
    if (s.plan.klass == KORCH_CLASS_REJECTED) return fail(KORCH_E_UNSUPPORTED, "rejected: " + s.plan.reject);
    std::string all;
    for (auto& v : s.plan.variants) all += "// variant: " + v.tag + "\n" + full_source(v) + "\n";
    return write_buf(all, buf, cap, needed);
  })
}

korch_status korch_compile(korch_graph* G, const int64_t* idx, int64_t n, int32_t threads, const char* cache_dir,
                           int32_t* ok) {
  if (!G || (n > 0 && !idx)) return fail(KORCH_E_ARG, "NULL argument");
  KORCH_TRY({
    std::vector<int64_t> v(idx, idx + n);
    for (auto i : v)
      if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
    std::string cd = cache_dir ? cache_dir : default_cache_dir();
    compile_many(G, v, threads, cd);
    bool all_ok = true;
    std::string first_err;
    for (int64_t k = 0; k < n; ++k) {
      const CandState& s = G->cs[v[k]];
      // a launch variant that fails to compile is dropped (the profiler skips it); the
      // candidate is generable while at least one variant compiled
      bool good = false;
      for (auto& var : s.plan.variants) {
        Module* m = G->ctx->module_for(var.name);
        if (m->compiled) good = true;
        else if (first_err.empty()) first_err = var.name + ": " + m->log;
      }
      if (ok) ok[k] = good ? 1 : 0;
      if (s.plan.klass != KORCH_CLASS_REJECTED && !good) all_ok = false;
    }
    if (!all_ok) return fail(KORCH_E_NVRTC, first_err);
    return KORCH_OK;
  })
}

korch_status korch_profile(korch_graph* G, const int64_t* idx, int64_t n, const korch_prof_opts* po, int64_t* cost) {
  if (!G || (n > 0 && (!idx || !cost))) return fail(KORCH_E_ARG, "NULL argument");
  KORCH_TRY({
    korch_ctx* ctx = G->ctx;
    ctx->bind();
    int warmup = po && po->warmup > 0 ? po->warmup : 3;
    int launches = po && po->launches > 0 ? po->launches : 20;
    int trials = po && po->trials > 0 ? po->trials : 5;
    bool flush = po && po->flush_l2;
    bool tune = !po || po->tune >= 0;
    int threads = po && po->compile_threads > 0 ? po->compile_threads : 0;
    std::vector<int64_t> v(idx, idx + n);
    for (auto i : v)
      if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
    compile_many(G, v, threads, default_cache_dir());
    CudaApi& cu = cuda();
    if (flush && !ctx->flush) {
      ctx->flush_bytes = std::max<size_t>((size_t)ctx->l2_bytes * 2, (size_t)256 << 20);
      CUresult r = cu.cuMemAlloc(&ctx->flush, ctx->flush_bytes);
      if (r != CUDA_SUCCESS) throw KorchError(KORCH_E_OOM, "flush buffer: " + cu_err(r));
    }
    CUevent e0, e1;
    prepare_fill(ctx);
    CU_CHECK(cu.cuEventCreate(&e0, CU_EVENT_DEFAULT));
    CU_CHECK(cu.cuEventCreate(&e1, CU_EVENT_DEFAULT));
    for (int64_t k = 0; k < n; ++k) {
      int64_t ci = v[k];
      CandState& s = G->cs[ci];
      cost[k] = INT64_MAX;
      if (s.plan.klass == KORCH_CLASS_REJECTED) { s.cost_ns = INT64_MAX; continue; }
      // Candidates whose generated kernels are identical (same source => same shapes,
      // strides and launch configuration) share one measurement.
      // variants to time: all of them when tuning; otherwise only the chosen one (the
      // first if none was chosen yet), and the choice is left as it is
      std::vector<int> vis;
      if (tune) for (int vi = 0; vi < (int)s.plan.variants.size(); ++vi) vis.push_back(vi);
      else vis.push_back(s.best >= 0 ? s.best : 0);
      const int keep_best = s.best;
      auto tkey = [&](int vi) {
        const KernelVariant& v = s.plan.variants[vi];
        return v.name + "|" + std::to_string(flush) + "|" + std::to_string(flush ? 1 : launches) + "|" +
               std::to_string(trials);
      };
      {
        bool all_cached = true;
        std::lock_guard<std::mutex> lk(ctx->mu);
        for (int vi : vis)
          if (!ctx->timings.count(tkey(vi))) all_cached = false;
        if (all_cached) {
          if (tune || s.var_ns.size() != s.plan.variants.size()) s.var_ns.assign(s.plan.variants.size(), -1);
          int64_t best = INT64_MAX;
          int bestv = -1;
          for (int vi : vis) {
            int64_t ns = ctx->timings[tkey(vi)];
            s.var_ns[vi] = ns;
            if (ns < best) { best = ns; bestv = vi; }
          }
          s.best = tune || keep_best < 0 ? bestv : keep_best;
          s.cost_ns = best;
          cost[k] = best;
          continue;
        }
      }
      // scratch buffers at the candidate's exact shapes (512 bytes of slack before the
      // first and after the last: a kernel's speculated boundary load stays mapped)
      std::vector<size_t> offs;
      size_t tot = 512;
      for (auto& r : s.plan.ext) {
        offs.push_back(tot);
        tot += ((size_t)tensor_bytes(G->g, r) + 255) & ~(size_t)255;
      }
      std::vector<size_t> out_offs;
      {
        std::vector<int> os{G->cands[ci].output};
        os.insert(os.end(), G->cands[ci].extra_outputs.begin(), G->cands[ci].extra_outputs.end());
        for (int o : os) {
          out_offs.push_back(tot);
          tot += ((size_t)tensor_bytes(G->g, Ref{false, o}) + 255) & ~(size_t)255;
        }
      }
      CUdeviceptr base = ctx->arena_get(tot + 512);
      std::vector<const void*> ins;
      for (size_t e = 0; e < s.plan.ext.size(); ++e) {
        const Ref& r = s.plan.ext[e];
        CUdeviceptr p = base + offs[e];
        size_t ne = (size_t)numel(G->g.shape_of(r));
        launch_fill(ctx, p, ne, G->g.dtype_of(r), (unsigned)(e + 1), ctx->pstream);
        ins.push_back((const void*)p);
      }
      std::vector<void*> outp;
      for (size_t oo : out_offs) outp.push_back((void*)(base + oo));
      int64_t best = INT64_MAX;
      int bestv = -1;
      if (tune || s.var_ns.size() != s.plan.variants.size()) s.var_ns.assign(s.plan.variants.size(), -1);
      for (int vi : vis) {
        Module* m = ctx->module_for(s.plan.variants[vi].name);
        if (!m->compiled) continue;
        try {
          int nl = flush ? 1 : launches;
          int ntr = trials;
          static const bool trace = getenv("KORCH_PROFILE_TRACE") != nullptr;
          if (trace) {
            std::fprintf(stderr, "[korch profile] cand %lld variant %d %s | %s\n", (long long)ci, vi,
                         s.plan.variants[vi].name.c_str(), s.plan.variants[vi].tag.c_str());
            std::fflush(stderr);
          }
          prepare_variant(ctx, s.plan.variants[vi]);
          {
            // one probe launch: slow kernels get fewer launches per graph / fewer trials
            // (the median over >= 3 trials of >= ~100 us of work stays stable)
            launch_variant(ctx, s.plan, vi, ins, outp, ctx->pstream);
            CU_CHECK(cu.cuEventRecord(e0, ctx->pstream));
            launch_variant(ctx, s.plan, vi, ins, outp, ctx->pstream);
            CU_CHECK(cu.cuEventRecord(e1, ctx->pstream));
            CU_CHECK(cu.cuEventSynchronize(e1));
            float ms = 0;
            CU_CHECK(cu.cuEventElapsedTime(&ms, e0, e1));
            if (!flush && ms > 0.005f) nl = std::max(1, std::min(nl, (int)(0.1f / ms)));
            if (ms > 0.2f) ntr = std::min(ntr, 3);
          }
          std::lock_guard<std::mutex> cap(ctx->capture_mu);
          CU_CHECK(cu.cuStreamBeginCapture(ctx->pstream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL));
          try {
            // launches after the first use programmatic dependent launch, as the executor
            // does for every kernel after a plan's first (A19: the executor's regime).
            // Cold-L2 timing: the flush, two event-record nodes and the kernel form one
            // graph, so the events bracket the kernel on the device with no host launch
            // latency in between.
            // (event records inside a capture must be EXTERNAL to become timestamped
            // event-record nodes instead of capture-internal dependencies)
            if (flush) {
              CU_CHECK(cu.cuMemsetD8Async(ctx->flush, 0x5a, ctx->flush_bytes, ctx->pstream));
              CU_CHECK(cu.cuEventRecordWithFlags(e0, ctx->pstream, CU_EVENT_RECORD_EXTERNAL));
            }
            for (int l = 0; l < nl; ++l) launch_variant(ctx, s.plan, vi, ins, outp, ctx->pstream, l > 0);
            if (flush) CU_CHECK(cu.cuEventRecordWithFlags(e1, ctx->pstream, CU_EVENT_RECORD_EXTERNAL));
          } catch (...) {
            CUgraph tmp;
            cu.cuStreamEndCapture(ctx->pstream, &tmp);
            if (tmp) cu.cuGraphDestroy(tmp);
            throw;
          }
          CUgraph graph;
          CU_CHECK(cu.cuStreamEndCapture(ctx->pstream, &graph));
          CUgraphExec ge;
          CU_CHECK(cu.cuGraphInstantiateWithFlags(&ge, graph, 0));
          cu.cuGraphDestroy(graph);
          for (int w = 0; w < (nl < launches ? 1 : warmup); ++w) CU_CHECK(cu.cuGraphLaunch(ge, ctx->pstream));
          std::vector<float> ts;
          for (int t = 0; t < ntr; ++t) {
            if (!flush) CU_CHECK(cu.cuEventRecord(e0, ctx->pstream));
            CU_CHECK(cu.cuGraphLaunch(ge, ctx->pstream));
            if (!flush) CU_CHECK(cu.cuEventRecord(e1, ctx->pstream));
            CU_CHECK(cu.cuEventSynchronize(e1));
            float ms = 0;
            CU_CHECK(cu.cuEventElapsedTime(&ms, e0, e1));
            ts.push_back(ms / nl);
          }
          cu.cuGraphExecDestroy(ge);
          std::sort(ts.begin(), ts.end());
          int64_t ns = (int64_t)std::llround((double)ts[ts.size() / 2] * 1e6);
          if (ns < 1) ns = 1;
          s.var_ns[vi] = ns;
          {
            std::lock_guard<std::mutex> lk(ctx->mu);
            ctx->timings[tkey(vi)] = ns;
          }
          if (ns < best) { best = ns; bestv = vi; }
        } catch (KorchError& e) {
          // a variant that fails to launch is rejected (cost = inf for it)
          g_err = e.what();
          CUresult r = cu.cuStreamSynchronize(ctx->pstream);
          if (r != CUDA_SUCCESS) { cu.cuEventDestroy(e0); cu.cuEventDestroy(e1); throw; }
        }
      }
      s.best = tune || keep_best < 0 ? bestv : keep_best;
      s.cost_ns = best;
      cost[k] = best;
    }
    cu.cuEventDestroy(e0);
    cu.cuEventDestroy(e1);
    return KORCH_OK;
  })
}

korch_status korch_variant_info(const korch_graph* G, int64_t i, int32_t* nv, int32_t* chosen, char* tag,
                                size_t cap) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
  const CandState& s = G->cs[i];
  if (nv) *nv = (int32_t)s.plan.variants.size();
  if (chosen) *chosen = s.best;
  if (tag && cap) {
    std::string t = s.plan.variants.empty() ? "rejected: " + s.plan.reject
                                            : s.plan.variants[s.best >= 0 ? s.best : 0].tag;
    size_t need;
    return write_buf(t, tag, cap, &need);
  }
  return KORCH_OK;
}

korch_status korch_variant_cost(const korch_graph* G, int64_t i, int32_t v, int64_t* ns) {
  if (!G || !ns) return fail(KORCH_E_ARG, "NULL argument");
  if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
  const CandState& s = G->cs[i];
  if (v < 0 || v >= (int32_t)s.plan.variants.size()) return fail(KORCH_E_ARG, "variant index out of range");
  *ns = v < (int32_t)s.var_ns.size() ? s.var_ns[v] : -1;
  return KORCH_OK;
}

korch_status korch_variant_name(const korch_graph* G, int64_t i, int32_t v, char* name, size_t cap, size_t* needed) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
  const CandState& s = G->cs[i];
  if (v < 0 || v >= (int32_t)s.plan.variants.size()) return fail(KORCH_E_ARG, "variant index out of range");
  return write_buf(s.plan.variants[v].name, name, cap, needed);
}

korch_status korch_select_variant(korch_graph* G, int64_t i, int32_t v) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
  CandState& s = G->cs[i];
  if (v < 0 || v >= (int32_t)s.plan.variants.size()) return fail(KORCH_E_ARG, "variant index out of range");
  s.best = v;
  return KORCH_OK;
}

korch_status korch_set_orchestration(korch_graph* G, const int64_t* sel, int64_t n, size_t* ws) {
  if (!G || (n > 0 && !sel)) return fail(KORCH_E_ARG, "NULL argument");
  KORCH_TRY({
    std::lock_guard<std::mutex> lk(G->mu);
    const Graph& g = G->g;
    std::vector<int64_t> order(sel, sel + n);
    for (auto i : order)
      if (i < 0 || i >= (int64_t)G->cands.size()) return fail(KORCH_E_ARG, "candidate index out of range");
    // A6: order by topological index of the output (the sink), ties by candidate index
    std::sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      int ta = g.topo_index[G->cands[a].output], tb = g.topo_index[G->cands[b].output];
      return ta != tb ? ta < tb : a < b;
    });
    auto outs_of = [&](int64_t i) {
      std::vector<int> os{G->cands[i].output};
      os.insert(os.end(), G->cands[i].extra_outputs.begin(), G->cands[i].extra_outputs.end());
      return os;
    };
    std::vector<int64_t> uniq;
    std::vector<int> producer(g.prims.size(), -1);  // prim -> step index of its first producer
    for (auto i : order) {
      bool any_new = false;
      for (int t : outs_of(i)) any_new = any_new || producer[t] < 0;
      if (!any_new) continue;  // A7: every output already bound to an earlier producer
      for (int t : outs_of(i))
        if (producer[t] < 0) producer[t] = (int)uniq.size();
      uniq.push_back(i);
    }
    // Eq. 4 / Eq. 4' (reading A32): every input of a kernel is materialised by a selected
    // kernel whose sink precedes its own; the first producer in order has the earliest sink
    for (size_t s = 0; s < uniq.size(); ++s)
      for (int p : G->cands[uniq[s]].inputs)
        if (producer[p] < 0 || g.topo_index[G->cands[uniq[producer[p]]].output] >= g.topo_index[G->cands[uniq[s]].output])
          return fail(KORCH_E_INFEASIBLE, "Eq. 4 violated: kernel " + std::to_string(uniq[s]) + " needs p" +
                                              std::to_string(p) + " which no earlier selected kernel produces");
    // Eq. 3: every output primitive is produced
    for (int t : g.outputs)
      if (producer[t] < 0) return fail(KORCH_E_INFEASIBLE, "Eq. 3 violated: output p" + std::to_string(t) + " not produced");
    for (auto i : uniq) {
      ensure_planned(G, i);
      if (G->cs[i].plan.klass == KORCH_CLASS_REJECTED)
        return fail(KORCH_E_NOT_SCHEDULABLE, "candidate " + std::to_string(i) + " is rejected: " + G->cs[i].plan.reject);
    }
    compile_many(G, uniq, 0, default_cache_dir());
    for (auto i : uniq) {
      const CandState& cs = G->cs[i];
      const KernelVariant& v = cs.plan.variants[cs.best >= 0 ? cs.best : 0];
      Module* m = G->ctx->module_for(v.name);
      if (!m->compiled) return fail(KORCH_E_NVRTC, v.name + ": " + m->log);
    }
    // liveness-based workspace plan
    std::vector<int> last_use(g.prims.size(), -1);
    for (size_t s = 0; s < uniq.size(); ++s)
      for (int p : G->cands[uniq[s]].inputs) last_use[p] = std::max(last_use[p], (int)s);
    std::map<int, int> out_index;
    for (size_t k = 0; k < g.outputs.size(); ++k)
      if (!out_index.count(g.outputs[k])) out_index[g.outputs[k]] = (int)k;
    struct Blk { size_t off, size; };
    std::vector<Blk> free_list;
    size_t top = 0;
    std::vector<size_t> off_of(g.prims.size(), 0);
    auto alloc = [&](size_t bytes) {
      bytes = (bytes + 255) & ~(size_t)255;
      for (size_t f = 0; f < free_list.size(); ++f)
        if (free_list[f].size >= bytes) {
          size_t o = free_list[f].off;
          free_list[f].off += bytes;
          free_list[f].size -= bytes;
          if (!free_list[f].size) free_list.erase(free_list.begin() + f);
          return o;
        }
      size_t o = top;
      top += bytes;
      return o;
    };
    auto release = [&](size_t off, size_t bytes) {
      bytes = (bytes + 255) & ~(size_t)255;
      free_list.push_back({off, bytes});
      std::sort(free_list.begin(), free_list.end(), [](const Blk& a, const Blk& b) { return a.off < b.off; });
      for (size_t f = 0; f + 1 < free_list.size();) {
        if (free_list[f].off + free_list[f].size == free_list[f + 1].off) {
          free_list[f].size += free_list[f + 1].size;
          free_list.erase(free_list.begin() + f + 1);
        } else ++f;
      }
    };
    std::vector<Step> steps;
    for (size_t s = 0; s < uniq.size(); ++s) {
      int64_t ci = uniq[s];
      CandState& cs = G->cs[ci];
      Step st;
      st.cand = (int)ci;
      st.variant = cs.best >= 0 ? cs.best : 0;
      for (auto& r : cs.plan.ext) {
        BufRef b;
        if (r.is_input) { b.kind = BufRef::Input; b.index = r.id; }
        else if (out_index.count(r.id)) { b.kind = BufRef::Output; b.index = out_index[r.id]; }
        else { b.kind = BufRef::Work; b.offset = off_of[r.id]; }
        st.args.push_back(b);
      }
      std::vector<std::pair<size_t, size_t>> scratch;  // (offset, bytes) released after this step
      for (int o : outs_of(ci)) {
        BufRef b;
        const size_t nb = (size_t)tensor_bytes(g, Ref{false, o});
        if (producer[o] != (int)s) {
          // a later producer of an already materialised tensor (A7) writes a dead copy
          b.kind = BufRef::Work;
          b.offset = alloc(nb);
          scratch.push_back({b.offset, nb});
        } else if (out_index.count(o)) {
          b.kind = BufRef::Output;
          b.index = out_index[o];
        } else {
          off_of[o] = alloc(nb);
          b.kind = BufRef::Work;
          b.offset = off_of[o];
          if (last_use[o] <= (int)s) scratch.push_back({b.offset, nb});  // never read again
        }
        st.outs.push_back(b);
      }
      // free tensors whose last consumer is this step
      for (int p : G->cands[ci].inputs)
        if (last_use[p] == (int)s && !out_index.count(p)) release(off_of[p], (size_t)tensor_bytes(g, Ref{false, p}));
      for (auto& sc : scratch) release(sc.first, sc.second);
      steps.push_back(st);
    }
    // step dependencies for concurrent replay (N4): step t follows step s < t when one
    // writes a buffer range the other reads or writes (workspace ranges are reused by the
    // liveness plan, so WAR / WAW matter as much as RAW)
    {
      struct Rg { int kind, idx; size_t lo, hi; };
      auto rg = [&](const BufRef& b, size_t nb) {
        if (b.kind == BufRef::Work) return Rg{2, 0, b.offset, b.offset + nb};
        return Rg{b.kind == BufRef::Output ? 1 : 0, b.index, 0, nb};
      };
      auto ov = [](const Rg& a, const Rg& b) { return a.kind == b.kind && a.idx == b.idx && a.lo < b.hi && b.lo < a.hi; };
      std::vector<std::vector<Rg>> rd(steps.size()), wr(steps.size());
      for (size_t t = 0; t < steps.size(); ++t) {
        const KernelPlan& kp = G->cs[steps[t].cand].plan;
        for (size_t a = 0; a < steps[t].args.size(); ++a)
          rd[t].push_back(rg(steps[t].args[a], (size_t)tensor_bytes(g, kp.ext[a])));
        std::vector<int> os = outs_of(steps[t].cand);
        for (size_t o = 0; o < steps[t].outs.size(); ++o)
          wr[t].push_back(rg(steps[t].outs[o], (size_t)tensor_bytes(g, Ref{false, os[o]})));
      }
      G->deps.assign(steps.size(), {});
      for (size_t t = 0; t < steps.size(); ++t)
        for (size_t s2 = 0; s2 < t; ++s2) {
          bool d = false;
          for (auto& w : wr[s2]) for (auto& r : rd[t]) d = d || ov(w, r);
          for (auto& r : rd[s2]) for (auto& w : wr[t]) d = d || ov(r, w);
          for (auto& w : wr[s2]) for (auto& w2 : wr[t]) d = d || ov(w, w2);
          // two launches of one kernel that owns a scratch buffer (module-wide) never overlap
          const KernelVariant& va = G->cs[steps[s2].cand].plan.variants[steps[s2].variant];
          const KernelVariant& vb = G->cs[steps[t].cand].plan.variants[steps[t].variant];
          d = d || (va.scratch_bytes > 0 && va.name == vb.name);
          if (d) G->deps[t].push_back((int)s2);
        }
    }
    G->steps = steps;
    G->ws_bytes = top;
    G->has_plan = true;
    if (G->gexec && cuda().ok) { cuda().cuGraphExecDestroy(G->gexec); G->gexec = nullptr; }
    if (G->gexec_host && cuda().ok) { cuda().cuGraphExecDestroy(G->gexec_host); G->gexec_host = nullptr; }
    G->cap_ptrs.clear();
    G->cap_ptrs_host.clear();
    if (ws) *ws = top;
    return KORCH_OK;
  })
}

korch_status korch_plan(const korch_graph* G, int64_t* nk, int64_t* order) {
  if (!G || !nk) return fail(KORCH_E_ARG, "NULL argument");
  if (!G->has_plan) return fail(KORCH_E_ARG, "no accepted orchestration");
  *nk = (int64_t)G->steps.size();
  if (order)
    for (size_t i = 0; i < G->steps.size(); ++i) order[i] = G->steps[i].cand;
  return KORCH_OK;
}

korch_status korch_execute(korch_graph* G, const void* const* inputs, void* const* outputs, void* workspace,
                           void* stream) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (!G->has_plan) return fail(KORCH_E_ARG, "no accepted orchestration (call korch_set_orchestration)");
  KORCH_TRY({
    korch_ctx* ctx = G->ctx;
    ctx->bind();
    CudaApi& cu = cuda();
    std::lock_guard<std::mutex> lk(G->mu);
    const Graph& g = G->g;
    std::vector<const void*> ptrs;
    for (size_t i = 0; i < g.inputs.size(); ++i) ptrs.push_back(inputs[i]);
    for (size_t i = 0; i < g.outputs.size(); ++i) ptrs.push_back(outputs[i]);
    ptrs.push_back(workspace);
    auto resolve = [&](const BufRef& b) -> void* {
      if (b.kind == BufRef::Input) return const_cast<void*>(inputs[b.index]);
      if (b.kind == BufRef::Output) return outputs[b.index];
      return static_cast<char*>(workspace) + b.offset;
    };
    auto resolve_outs = [&](const Step& st) {
      std::vector<void*> r;
      for (auto& b : st.outs) r.push_back(resolve(b));
      return r;
    };
    static const bool direct = getenv("KORCH_EXEC_DIRECT") != nullptr;
    static const bool use_pdl = !(getenv("KORCH_PDL") && std::string(getenv("KORCH_PDL")) == "0");
    if (direct || !G->gexec || ptrs != G->cap_ptrs)
      for (auto& st : G->steps) prepare_variant(ctx, G->cs[st.cand].plan.variants[st.variant]);
    if (direct) {  // plain stream launches (profilers that cannot follow graph replays)
      for (auto& st : G->steps) {
        std::vector<const void*> ins;
        for (auto& a : st.args) ins.push_back(resolve(a));
        launch_variant(ctx, G->cs[st.cand].plan, st.variant, ins, resolve_outs(st), (CUstream)stream);
      }
      return KORCH_OK;
    }
    if (!G->gexec || ptrs != G->cap_ptrs) {
      if (G->gexec) { cu.cuGraphExecDestroy(G->gexec); G->gexec = nullptr; }
      std::lock_guard<std::mutex> cap(ctx->capture_mu);
      CU_CHECK(cu.cuStreamBeginCapture(ctx->pstream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL));
      try {
        // every kernel after the first of its stream overlaps its prologue with its
        // predecessor (PDL)
        capture_steps(ctx, G, use_pdl, [&](const Step& st, CUstream sm, bool pdl) {
          std::vector<const void*> ins;
          for (auto& a : st.args) ins.push_back(resolve(a));
          launch_variant(ctx, G->cs[st.cand].plan, st.variant, ins, resolve_outs(st), sm, pdl);
        });
      } catch (...) {
        CUgraph tmp = nullptr;
        cu.cuStreamEndCapture(ctx->pstream, &tmp);
        if (tmp) cu.cuGraphDestroy(tmp);
        throw;
      }
      CUgraph graph;
      CU_CHECK(cu.cuStreamEndCapture(ctx->pstream, &graph));
      CU_CHECK(cu.cuGraphInstantiateWithFlags(&G->gexec, graph, 0));
      cu.cuGraphDestroy(graph);
      G->cap_ptrs = ptrs;
    }
    CU_CHECK(cu.cuGraphLaunch(G->gexec, (CUstream)stream));
    return KORCH_OK;
  })
}

// Host <-> device transfers of korch_execute_host as a kernel: page-locked host memory is
// mapped into the device's unified address space, so 16-byte loads/stores over the
// host link replace copy-engine memcpy nodes (whose per-copy set-up dominates at the
// ~100 KB sizes of a bs-1 inference).  Falls back to memcpy nodes when a buffer is not
// device-accessible or not 16-byte aligned.
static const KernelVariant& copy_variant() {
  static KernelVariant v = [] {
    KernelVariant k;
    k.name = "korch_copy16_v1";
    k.block = 256;
    k.source =
        "extern \"C\" __global__ void __launch_bounds__(256) korch_copy16_v1(const uint4* __restrict__ src, "
        "uint4* __restrict__ dst, unsigned long long n16) {\n"
        "  pdl_trigger();\n  pdl_wait();\n"
        "  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n16; i += gridDim.x * 256ull)\n"
        "    dst[i] = src[i];\n}\n";
    return k;
  }();
  return v;
}

// Above this size host<->device transfers use copy-engine memcpy nodes (DMA at full link
// bandwidth) instead of copy kernels / kernel stores over mapped host memory.
static const size_t kHostKernelCopyMax = 1u << 20;

static bool launch_copy(korch_ctx* ctx, const void* src, void* dst, size_t bytes, CUstream stream, bool pdl) {
  CudaApi& cu = cuda();
  if (((unsigned long long)src | (unsigned long long)dst | bytes) & 15) return false;
  if (bytes > kHostKernelCopyMax) return false;
  CUdeviceptr ds = 0, dd = 0;
  if (cu.cuPointerGetAttribute(&ds, CU_POINTER_ATTRIBUTE_DEVICE_POINTER, (CUdeviceptr)src) != CUDA_SUCCESS) return false;
  if (cu.cuPointerGetAttribute(&dd, CU_POINTER_ATTRIBUTE_DEVICE_POINTER, (CUdeviceptr)dst) != CUDA_SUCCESS) return false;
  const KernelVariant& v = copy_variant();
  Module* m = ctx->module_for(v.name);
  if (!m->compiled || !m->fn) return false;  // prepare_copy() runs before stream capture
  CUfunction fn = m->fn;
  unsigned long long n16 = bytes / 16;
  unsigned grid = (unsigned)std::max<unsigned long long>(1, std::min<unsigned long long>(4 * 148, (n16 + 255) / 256));
  void* args[] = {&ds, &dd, &n16};
  CUlaunchConfig cfg{};
  cfg.gridDimX = grid;
  cfg.gridDimY = cfg.gridDimZ = 1;
  cfg.blockDimX = 256;
  cfg.blockDimY = cfg.blockDimZ = 1;
  cfg.hStream = stream;
  CUlaunchAttribute at[1];
  at[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
  at[0].value.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  CU_CHECK(cu.cuLaunchKernelEx(&cfg, fn, args, nullptr));
  return true;
}

// compile (cached) and load the copy kernel; must run outside stream capture
static void prepare_copy(korch_ctx* ctx) {
  const KernelVariant& v = copy_variant();
  Module* m = ctx->module_for(v.name);
  if (!m->compiled && !m->failed) compile_batch({{m, &v}}, default_cache_dir());
  if (m->compiled) load_fn(ctx, m, v);
}

korch_status korch_execute_host(korch_graph* G, const void* const* host_inputs, const void* const* dev_inputs,
                                void* const* host_outputs, void* const* dev_outputs, void* workspace, void* stream) {
  if (!G) return fail(KORCH_E_ARG, "NULL graph");
  if (!host_inputs || !dev_inputs || !host_outputs || !dev_outputs) return fail(KORCH_E_ARG, "NULL pointer array");
  if (!G->has_plan) return fail(KORCH_E_ARG, "no accepted orchestration (call korch_set_orchestration)");
  KORCH_TRY({
    korch_ctx* ctx = G->ctx;
    ctx->bind();
    CudaApi& cu = cuda();
    std::lock_guard<std::mutex> lk(G->mu);
    const Graph& g = G->g;
    std::vector<const void*> ptrs;
    for (size_t i = 0; i < g.inputs.size(); ++i) { ptrs.push_back(host_inputs[i]); ptrs.push_back(dev_inputs[i]); }
    for (size_t i = 0; i < g.outputs.size(); ++i) { ptrs.push_back(host_outputs[i]); ptrs.push_back(dev_outputs[i]); }
    ptrs.push_back(workspace);
    // Outputs whose host buffer is mapped into the device's address space (page-locked,
    // 16-byte aligned) are written by their producing kernel straight into host memory:
    // no device output buffer, no D2H copy.
    static const bool ce_only = getenv("KORCH_E2E_MEMCPY") != nullptr;
    std::vector<void*> direct_out(g.outputs.size(), nullptr);
    // ... unless a kernel of the plan also reads that output (its consumers would then
    // read, or build TMA maps over, system memory across the host link)
    std::vector<bool> read_in_plan(g.outputs.size(), false);
    for (auto& st : G->steps)
      for (auto& a : st.args)
        if (a.kind == BufRef::Output) read_in_plan[a.index] = true;
    for (size_t j = 0; j < g.outputs.size(); ++j) {
      CUdeviceptr d = 0;
      // (small outputs only: a kernel's scattered stores over the host link run far below
      // the copy engine's bandwidth once the output is more than a few hundred KB)
      if (!ce_only && !read_in_plan[j] && host_outputs[j] && ((unsigned long long)host_outputs[j] & 15) == 0 &&
          (size_t)tensor_bytes(g, Ref{false, g.outputs[j]}) <= kHostKernelCopyMax &&
          cu.cuPointerGetAttribute(&d, CU_POINTER_ATTRIBUTE_DEVICE_POINTER, (CUdeviceptr)host_outputs[j]) ==
              CUDA_SUCCESS)
        direct_out[j] = (void*)d;
    }
    auto resolve = [&](const BufRef& b) -> void* {
      if (b.kind == BufRef::Input) return const_cast<void*>(dev_inputs[b.index]);
      if (b.kind == BufRef::Output) return direct_out[b.index] ? direct_out[b.index] : dev_outputs[b.index];
      return static_cast<char*>(workspace) + b.offset;
    };
    auto resolve_outs = [&](const Step& st) {
      std::vector<void*> r;
      for (auto& b : st.outs) r.push_back(resolve(b));
      return r;
    };
    static const bool use_pdl = !(getenv("KORCH_PDL") && std::string(getenv("KORCH_PDL")) == "0");
    if (!G->gexec_host || ptrs != G->cap_ptrs_host) {
      for (auto& st : G->steps) prepare_variant(ctx, G->cs[st.cand].plan.variants[st.variant]);
      prepare_copy(ctx);
      if (G->gexec_host) { cu.cuGraphExecDestroy(G->gexec_host); G->gexec_host = nullptr; }
      std::lock_guard<std::mutex> cap(ctx->capture_mu);
      CU_CHECK(cu.cuStreamBeginCapture(ctx->pstream, CU_STREAM_CAPTURE_MODE_THREAD_LOCAL));
      try {
        bool any = false;  // a copy kernel was launched before this one (PDL between copies)
        for (size_t i = 0; i < g.inputs.size(); ++i)
          if (host_inputs[i]) {
            const size_t nb = (size_t)tensor_bytes(g, Ref{true, (int)i});
            if (ce_only || !launch_copy(ctx, host_inputs[i], const_cast<void*>(dev_inputs[i]), nb, ctx->pstream,
                                        use_pdl && any))
              CU_CHECK(cu.cuMemcpyHtoDAsync((CUdeviceptr)dev_inputs[i], host_inputs[i], nb, ctx->pstream));
            any = true;
          }
        // the first plan kernel of every stream is launched WITHOUT programmatic
        // serialisation: plan kernels fetch graph inputs (weights, residual tiles, a staged
        // LayerNorm input) before griddepcontrol.wait, and here the inputs are being written
        // by the copy kernels just launched, so the plan may only start once they completed
        capture_steps(ctx, G, use_pdl, [&](const Step& st, CUstream sm, bool pdl) {
          std::vector<const void*> ins;
          for (auto& a : st.args) ins.push_back(resolve(a));
          launch_variant(ctx, G->cs[st.cand].plan, st.variant, ins, resolve_outs(st), sm, pdl);
        });
        for (size_t j = 0; j < g.outputs.size(); ++j)
          if (host_outputs[j] && !direct_out[j]) {
            const size_t nb = (size_t)tensor_bytes(g, Ref{false, g.outputs[j]});
            if (ce_only || !launch_copy(ctx, dev_outputs[j], host_outputs[j], nb, ctx->pstream, use_pdl))
              CU_CHECK(cu.cuMemcpyDtoHAsync(host_outputs[j], (CUdeviceptr)dev_outputs[j], nb, ctx->pstream));
          }
      } catch (...) {
        CUgraph tmp = nullptr;
        cu.cuStreamEndCapture(ctx->pstream, &tmp);
        if (tmp) cu.cuGraphDestroy(tmp);
        throw;
      }
      CUgraph graph;
      CU_CHECK(cu.cuStreamEndCapture(ctx->pstream, &graph));
      CU_CHECK(cu.cuGraphInstantiateWithFlags(&G->gexec_host, graph, 0));
      cu.cuGraphDestroy(graph);
      G->cap_ptrs_host = ptrs;
    }
    CU_CHECK(cu.cuGraphLaunch(G->gexec_host, (CUstream)stream));
    return KORCH_OK;
  })
}

}  // extern "C"
