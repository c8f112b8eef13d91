/*
 * korch.h — C ABI of the B200-native Korch hot path (arXiv 2406.09465).
 *
 * The calls follow the paper's statement of the problem:
 *   load a primitive graph G=(P,E)
 *   enumerate candidate kernels (Alg. 1, Theorem 1)
 *   profile each candidate's cost c_i (PROFILING, inf on failure)
 *   accept an orchestration u (Eq. 3/4 checked)
 *   execute it (sequential stitched kernels)
 * The BLP itself (Eq. 2-4 optimisation) is NOT in this library: the caller
 * solves it and passes the selection to korch_set_orchestration.
 *
 * Conventions
 *   - Every function returns korch_status (0 = KORCH_OK, negative = error) and
 *     never throws across the ABI; korch_last_error() returns a thread-local,
 *     NUL-terminated message describing the last failure on this thread.
 *   - The library owns korch_ctx, korch_graph, candidate tables and the
 *     compiled kernels.  The caller owns every device buffer: graph inputs
 *     (activations AND weights), outputs and the workspace.  Buffers are
 *     row-major, contiguous, in the dtype declared in the graph JSON ("f32"
 *     = IEEE float, "bf16" = bfloat16 bits), 16-byte aligned.
 *   - Pointers returned inside korch_cand_desc stay valid until the graph is
 *     freed or re-enumerated.
 *   - NaN/Inf propagate per IEEE; division by zero is not an error.
 *   - No allocation happens inside korch_execute.
 */
#ifndef KORCH_H_
#define KORCH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t korch_status;

#define KORCH_OK                 0
#define KORCH_E_ARG             -1  /* bad argument (NULL, out of range, wrong state)      */
#define KORCH_E_PARSE           -2  /* malformed graph JSON                                 */
#define KORCH_E_SHAPE           -3  /* shape inference failed                               */
#define KORCH_E_CYCLE           -4  /* graph is not a DAG                                   */
#define KORCH_E_STATE_EXPLOSION -5  /* more execution states than opts.max_states           */
#define KORCH_E_INFEASIBLE      -6  /* selection violates Eq. 3 or Eq. 4                    */
#define KORCH_E_NOT_SCHEDULABLE -7  /* selection contains a rejected (cost = inf) kernel    */
#define KORCH_E_NVRTC           -8  /* runtime compilation of a kernel failed               */
#define KORCH_E_CUDA            -9  /* CUDA driver error (or no driver / no device)         */
#define KORCH_E_OOM            -10  /* device allocation failed                             */
#define KORCH_E_UNSUPPORTED    -11  /* operator / primitive without a rule or template      */

/* Template classes (SURVEY.md §8(a') "template acceptance"). */
#define KORCH_CLASS_REJECTED  0     /* no template can generate it: cost = inf      */
#define KORCH_CLASS_PW        1     /* elementwise / broadcast / layout                     */
#define KORCH_CLASS_RR        2     /* row reduce -> broadcast                              */
#define KORCH_CLASS_GEMM      3     /* one dense linear primitive + fused views/epilogue    */

typedef struct korch_ctx korch_ctx;
typedef struct korch_graph korch_graph;

/* Options for korch_enumerate. Zero-initialised fields take the defaults. */
typedef struct {
  int32_t max_prims;          /* reject candidates with more primitives; default 16 */
  int32_t keep_multi_linear;  /* 1 = keep candidates with >= 2 dense linear prims; default 0 */
  int64_t max_states;         /* KORCH_E_STATE_EXPLOSION above this; default 1,000,000       */
  int32_t partition_max;      /* > 0: partition (reading A17) into parts of about this
                                 many primitives; 0: only graphs > 256 primitives, parts of 64 */
  int32_t attention_pairs;    /* 1: keep candidates with two MatMuls where the first feeds the
                                 second's A operand (fused attention; NEXT item N2) */
  int32_t max_outputs;        /* N1 ("for O in P'"; reading A32):
                                 <= 1: single-output candidates only (default); k > 1 (capped
                                 at 4): every single-output candidate (P', o) also yields
                                 (P', o, E) for each non-empty E of at most k - 1 members of
                                 P' other than o that have a consumer outside P' (or are graph
                                 outputs) and o's shape; E is materialised too            */
} korch_enum_opts;

/* One candidate kernel (P', o): a convex set with a unique sink o (reading A4). */
typedef struct {
  int32_t n_members;          /* |P'|                                                       */
  const int32_t* members;     /* primitive ids, ascending                                   */
  int32_t output;             /* o: the single materialised output primitive    */
  int32_t n_inputs;           /* primitive inputs: ids outside P' feeding P' (I row) */
  const int32_t* inputs;      /* ascending                                                  */
  int32_t n_graph_inputs;     /* graph-input tensors read by the kernel                     */
  const int32_t* graph_inputs;/* indices into the graph's "inputs" list, ascending          */
  int32_t klass;              /* KORCH_CLASS_*                                              */
  int32_t n_dense_linear;     /* dense linear primitives inside (reading A18)               */
  int64_t bytes;              /* algorithmic HBM bytes: external inputs read + output       */
  double flops;               /* 2*M*N*K summed over dense linear members                   */
  const char* signature;      /* canonical text of the generated kernel (dedup key)         */
  int32_t part;               /* partition part the candidate lies in (0 if unpartitioned)  */
  int32_t n_extra_outputs;    /* |E|: secondary materialised outputs (N1, reading A32)      */
  const int32_t* extra_outputs;/* primitive ids, ascending; the kernel writes them after o    */
} korch_cand_desc;

/* Options for korch_profile (reading A19). Zero-initialised fields take the defaults. */
typedef struct {
  int32_t warmup;             /* untimed graph replays before timing; default 3            */
  int32_t launches;           /* back-to-back launches captured per CUDA graph; default 20 */
  int32_t trials;             /* timed replays; median is reported; default 5              */
  int32_t flush_l2;           /* 1 = overwrite a >L2 buffer before every trial             */
  int32_t compile_threads;    /* parallel NVRTC jobs; default = hardware threads           */
  int32_t tune;               /* >= 0: time every launch variant, keep the fastest; -1: first only */
} korch_prof_opts;

/* Library version string, e.g. "korch-b200 0.1". */
const char* korch_version(void);

/* Thread-local message of the last failing call on this thread (never NULL). */
const char* korch_last_error(void);

/* Create a context.  cuda_device >= 0 binds that device's primary context
 * (shared with PyTorch); cuda_device = -1 creates a host-only context that can
 * load, enumerate and generate/compile kernels but not profile or execute
 * (returns KORCH_E_CUDA for those).  Errors: KORCH_E_CUDA if the driver or the
 * device is missing. */
korch_status korch_create(int32_t cuda_device, korch_ctx** out);
korch_status korch_destroy(korch_ctx* ctx);

/* Parse a graph JSON of n bytes (schema in korch_workloads/graphs.py; SPEC
 * S:131-135 plus "dtype").  Level "operator" runs the fission rules (
 * DESIGN.md readings A9-A16); level "primitive" is taken as is.  Shapes are
 * inferred; the graph must be a DAG.  Errors: KORCH_E_PARSE, KORCH_E_SHAPE,
 * KORCH_E_CYCLE, KORCH_E_UNSUPPORTED. */
korch_status korch_graph_load(korch_ctx* ctx, const char* json, size_t n, korch_graph** out);
korch_status korch_graph_free(korch_graph* g);

/* Sizes of the loaded primitive graph. */
korch_status korch_graph_info(const korch_graph* g, int32_t* n_prims, int32_t* n_inputs,
                              int32_t* n_outputs);

/* Write the primitive graph as JSON (level "primitive") into buf (capacity cap,
 * NUL-terminated).  *needed receives the full length + 1; if cap is too small
 * the call writes nothing and returns KORCH_E_ARG. */
korch_status korch_graph_dump(const korch_graph* g, char* buf, size_t cap, size_t* needed);

/* Structural validation report ("ok" or one violation per line); violations are
 * data, not failures. */
korch_status korch_validate(const korch_graph* g, char* report, size_t cap);

/* Alg. 1 with the empty state seeded (reading A1): DFS over
 * execution states, candidates = D2 \ D1 with a unique sink (A3/A4), pruned
 * and classified into templates.  Candidates are in canonical order
 * (output id, popcount, member ids).  Errors: KORCH_E_STATE_EXPLOSION. */
korch_status korch_enumerate(korch_graph* g, const korch_enum_opts* opts, int64_t* n_cands,
                             int64_t* n_states);

/* Describe candidate i (0 <= i < n_cands). */
korch_status korch_candidate(const korch_graph* g, int64_t i, korch_cand_desc* out);

/* Generated CUDA source of candidate i (for inspection); same buffer protocol
 * as korch_graph_dump.  Rejected candidates yield KORCH_E_UNSUPPORTED. */
korch_status korch_candidate_source(korch_graph* g, int64_t i, char* buf, size_t cap,
                                    size_t* needed);

/* Generate and compile (NVRTC, -arch=sm_100a) candidates idx[0..n).  Works on
 * host-only contexts (no GPU needed).  cache_dir (may be NULL) holds cubins keyed
 * by source hash.  ok[k] (caller-owned, n entries, may be NULL) = 1 when at least
 * one launch variant of candidate idx[k] compiled (variants that fail are dropped).
 * Returns KORCH_E_NVRTC (message = first compiler log) when a generable candidate
 * has no compiled variant; ok[] is filled either way. */
korch_status korch_compile(korch_graph* g, const int64_t* idx, int64_t n, int32_t threads,
                           const char* cache_dir, int32_t* ok);

/* PROFILING(P', O) of candidates idx[0..n) on the context's device: compile if
 * needed, time launches on seeded scratch inputs at the candidate's exact
 * shapes, write the median per-launch time in integer nanoseconds to cost_ns[k]
 * (caller-owned, n entries); INT64_MAX = cannot be generated (infinity). */
korch_status korch_profile(korch_graph* g, const int64_t* idx, int64_t n,
                           const korch_prof_opts* opts, int64_t* cost_ns);

/* Launch variants of candidate i (tile / thread-group configurations of its
 * template; the profiler keeps the fastest).  *n_variants and *chosen (-1 = not
 * profiled yet, variant 0 is used) may be NULL; tag receives the chosen (or
 * first) variant's description, same buffer protocol as korch_graph_dump. */
korch_status korch_variant_info(const korch_graph* g, int64_t i, int32_t* n_variants, int32_t* chosen,
                                char* tag, size_t cap);

/* Profiled median time of launch variant v of candidate i in integer ns (-1 if it
 * was not profiled, INT64_MAX if it failed to launch). */
korch_status korch_variant_cost(const korch_graph* g, int64_t i, int32_t v, int64_t* ns);

/* Kernel (entry-point) name of launch variant v of candidate i: a hash of the kernel's
 * generated source, i.e. of everything that determines what it computes and how it is
 * launched (with the shared prelude fixed; see korch_version).  Used as the key of
 * profiled costs in a tuning database.  Same buffer protocol as
 * korch_graph_dump; KORCH_E_ARG if i or v is out of range. */
korch_status korch_variant_name(const korch_graph* g, int64_t i, int32_t v, char* name, size_t cap,
                                size_t* needed);

/* Force candidate i to use launch variant v (e.g. to replay a plan without
 * re-profiling).  Takes effect at the next korch_set_orchestration. */
korch_status korch_select_variant(korch_graph* g, int64_t i, int32_t v);

/* Accept a selection u (sel[0..n) candidate indices with u_i = 1).  Checks Eq. 3
 * and Eq. 4 (KORCH_E_INFEASIBLE), that no member was rejected
 * (KORCH_E_NOT_SCHEDULABLE); orders kernels by the topological index of their
 * output (reading A6; duplicates keep the earliest, A7); plans intermediate
 * buffers by liveness; *workspace_bytes = device bytes the caller must provide
 * to korch_execute. */
korch_status korch_set_orchestration(korch_graph* g, const int64_t* sel, int64_t n,
                                     size_t* workspace_bytes);

/* Number of kernels in the accepted plan and their candidate indices in launch
 * order (order may be NULL; otherwise it must hold *n_kernels entries). */
korch_status korch_plan(const korch_graph* g, int64_t* n_kernels, int64_t* order);

/* Execute the accepted orchestration asynchronously on `stream` (a CUstream /
 * cudaStream_t; NULL = legacy default stream).  inputs[i] = device pointer of
 * graph input i (order of the JSON "inputs"), outputs[j] = device pointer of
 * output j (order of "outputs"), workspace = >= workspace_bytes device bytes.
 * The kernel sequence is captured once into a CUDA graph per distinct pointer
 * set and replayed.  Errors: KORCH_E_ARG (no plan), KORCH_E_CUDA. */
korch_status korch_execute(korch_graph* g, const void* const* inputs, void* const* outputs,
                           void* workspace, void* stream);

/* End-to-end execution with host buffers (the user-facing call of an inference
 * service: P:456-459's execution plus the transfers around it).  For every graph
 * input i with host_inputs[i] != NULL, numel*dtype bytes are copied host -> device
 * into dev_inputs[i] (inputs with a NULL host pointer, e.g. resident weights, are
 * used in place); the accepted orchestration then runs exactly as in
 * korch_execute; then every output j with host_outputs[j] != NULL is copied
 * device -> host from dev_outputs[j] -- or, when host_outputs[j] is page-locked,
 * mapped and 16-byte aligned, written there directly by the kernel producing it
 * (dev_outputs[j] is then left untouched).  Copies and kernels are captured into one
 * CUDA graph per distinct pointer set and replayed asynchronously on `stream`;
 * host buffers should be page-locked (pinned) for the copies to be asynchronous.
 * The caller owns all buffers.  Errors: KORCH_E_ARG (no plan / NULL arrays),
 * KORCH_E_CUDA. */
korch_status korch_execute_host(korch_graph* g, const void* const* host_inputs,
                                const void* const* dev_inputs, void* const* host_outputs,
                                void* const* dev_outputs, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KORCH_H_ */
