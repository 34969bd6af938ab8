/* stitch_b200.h — the C-ABI boundary of the B200 stitched-kernel executor.
 *
 * The reference (arXiv 2009.10924 artifact, /root/reference/proj) is a C++
 * library with no FFI of its own; its public entry points for this path are
 * the C++ functions named below.  These extern "C" functions are what a
 * binding to that path binds (ctypes in paper_2009_10924_b200/stitch.py; a
 * cgo/JNI/N-API stub would bind the same symbols).
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.
 *
 * Conventions: every int-returning call returns 0 on success, nonzero on
 * failure with a message in stc_last_error() (thread-local).  Codes:
 * 1 = parse/config/planner error, 2 = execution fault / compare mismatch,
 * 3 = CUDA/NVRTC error, 4 = bad argument.  Strings returned through char**
 * are malloc'd; release them with stc_free().  Handles are owned by the
 * caller and released with the matching *_destroy().  A stc_exec is bound to
 * one GPU and must be driven by one host thread at a time (one process or
 * thread per GPU for multi-GPU use).
 */
#ifndef STITCH_B200_H
#define STITCH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stc_graph stc_graph; /* stitch::CompGraph */
typedef struct stc_plan stc_plan;   /* FusionPlan + per-pattern KernelPlan + MachineModel */
typedef struct stc_exec stc_exec;   /* compiled plan on one GPU: cubins, buffers, CUDA Graph */

enum { STC_F32 = 0, STC_F16 = 1, STC_I32 = 2, STC_BOOL = 3 }; /* stitch::DType order */

const char* stc_last_error(void);
void stc_free(void* p);
const char* stc_version(void);

/* ---- graph IR ------------------------------------------------------------
 * replaces stitch::parse_graph / serialize_graph
 * (/root/reference/proj/include/stitch/parser.hpp:21-25, src/parser.cpp:162-285) */
int stc_graph_parse(const char* text, stc_graph** out);
void stc_graph_destroy(stc_graph* g);
int stc_graph_serialize(const stc_graph* g, char** out);
int stc_graph_num_nodes(const stc_graph* g);
/* which: 0 = parameters (declaration order), 1 = graph outputs (output order).
 * Returns the count; with i >= 0 also fills name/dtype/rank/dims[8]. */
int stc_graph_io(const stc_graph* g, int which, int i, const char** name, int* dtype, int* rank,
                 int64_t* dims);

/* ---- planning ------------------------------------------------------------
 * replaces stitch::explore_fusion_plan + CostModels::plan_for + plan_to_json
 * (include/stitch/explorer.hpp:74-75, explorer.hpp:36, src/pipeline.cpp:45-78,
 *  the body of run_pipeline src/pipeline.cpp:124-146).
 * cfg_path NULL/"" -> $STITCH_DEVICE_CONFIG or built-in defaults; k/beam <= 0
 * keep the cfg's values. */
int stc_plan_create(const stc_graph* g, const char* cfg_path, int k, int beam, stc_plan** out);
/* explicit patterns (vertex ids; pattern p = verts[offs[p] .. offs[p+1]-1]),
 * each planned with stitch::plan_kernel (include/stitch/planner.hpp:101-103);
 * rc 1 if a pattern is infeasible */
int stc_plan_from_patterns(const stc_graph* g, const char* cfg_path, const int* verts,
                           const int* offs, int n_patterns, stc_plan** out);
void stc_plan_destroy(stc_plan* p);
int stc_plan_json(const stc_plan* p, uint64_t seed, char** out);
int stc_plan_num_patterns(const stc_plan* p);
/* pattern i: vertex ids (up to cap) -> count; program text via kernel_text */
int stc_plan_pattern(const stc_plan* p, int i, int* verts, int cap);
int stc_plan_kernel_text(const stc_plan* p, int i, char** out);
/* NON-PARITY refinement: after the reference explorer,
 * greedily merge launch units along graph edges whenever the merge saves HBM
 * bytes or a launch and the merged pattern is plannable (reference
 * plan_kernel) and expressible by a stitching template.  The plan then no
 * longer equals the reference's; plan.json / kernel texts follow it. */
int stc_plan_refine(stc_plan* p, int* merges, int64_t* bytes_saved);
/* the last refinement's search effort: feasibility probes spent and whether
 * the deterministic probe budget (STITCH_REFINE_MAX_PROBES, default 2000)
 * stopped it before convergence (the refined plan is then a prefix of the
 * converged one -- never host-speed dependent) */
int stc_plan_refine_info(const stc_plan* p, int64_t* probes, int* budget_hit);
int stc_plan_stats(const stc_plan* p, int* stitched_kernels, int* baseline_kernels,
                   int64_t* delta_evaluate_calls);
/* stitch::plan_kernel on one vertex set -> program text; rc 1 = infeasible */
int stc_plan_kernel(const stc_graph* g, const char* cfg_path, const int* verts, int n,
                    char** program_text);

/* ---- execution on B200 ---------------------------------------------------
 * replaces stitch::eval_plan / run_program / eval_reference
 * (include/stitch/sim.hpp:33-47, src/sim.cpp:231-514): the reference walks
 * the plan on a CPU SIMT interpreter; here every planned pattern is one
 * NVRTC-compiled sm_100a kernel, uncovered fusable ops are singleton kernels,
 * opaque ops a placeholder kernel, all replayed as ONE CUDA Graph. */
enum {
  STC_EXEC_STITCHED = 0, /* dataflow templates (local/regional/global/independent) */
  STC_EXEC_PROGRAM = 1,  /* translate each planned abstract program statement for statement */
  STC_EXEC_UNFUSED = 2,  /* one kernel per op: eval_reference semantics on the GPU */
  STC_EXEC_NO_GRAPH = 8, /* flag: plain stream launches instead of a CUDA Graph */
  STC_EXEC_GEMM = 16     /* flag (model mode, non-parity): opaque_compute ops shaped like a matmul
                            A[..,M,K].B[K,N] run as cuBLASLt GEMMs (TF32 tensor cores; STITCH_GEMM_FP32=1
                            for full f32) instead of the reference's mean-of-operands placeholder */
};
/* code generation only (no device needed): the plan's CUDA module source and
 * a JSON description of its kernels */
int stc_codegen(const stc_plan* p, int mode, char** cuda_source, char** kernels_json);
int stc_exec_create(const stc_plan* p, int device, int mode, stc_exec** out);
/* Asynchronous compilation (the paper's async mode): returns
 * as soon as code generation is done; NVRTC runs on a worker thread.
 * stc_exec_ready() polls (1 = compiled), stc_exec_wait() blocks; every
 * execution call waits implicitly. */
int stc_exec_create_async(const stc_plan* p, int device, int mode, stc_exec** out);
int stc_exec_ready(const stc_exec* e);
int stc_exec_wait(stc_exec* e);
/* Persistent cubin-cache warm-up: generate and NVRTC-compile the modules of n
 * plans on `threads` host threads (no GPU needed), so later stc_exec_create
 * calls are cache hits.  *compiled / *cached: modules built now / found. */
int stc_cache_warm(const stc_plan* const* plans, int n, int mode, int threads, int* compiled, int* cached);
void stc_exec_destroy(stc_exec* e);
int stc_exec_num_kernels(const stc_exec* e);
/* JSON array: per launched kernel {name, template, pattern, grid, block, smem, bytes} */
int stc_exec_describe(const stc_exec* e, char** json);
int stc_exec_source(const stc_exec* e, char** cuda_source);
/* end to end with HOST buffers: H2D of every parameter, graph launch, D2H of
 * every output, synchronise.  Buffers hold the tensor's dtype natively
 * (f32 / f16 bits / i32 / u8 bool), parameters and outputs in stc_graph_io order. */
int stc_exec_run_host(stc_exec* e, const void* const* inputs, void* const* outputs);
/* Pipelined host execution of a batch `nchunks` times larger than the
 * executor's graph (build `e` from the chunk graph, e.g. batch 32/8):
 * inputs[i] holds nchunks consecutive chunks when input_chunked[i] != 0
 * (NULL = all chunked), else one tensor shared by every chunk; outputs[i]
 * receives nchunks consecutive chunks.  H2D of chunk k+1, the plan's graph
 * on chunk k and D2H of chunk k-1 overlap (separate copy-engine streams).
 * Same result as nchunks calls of stc_exec_run_host on the slices. */
int stc_exec_run_host_chunked(stc_exec* e, const void* const* inputs, void* const* outputs, int nchunks,
                              const int* input_chunked);
/* Zero-copy host execution: every input/output buffer must be pinned host
 * memory mapped into the device address space (cudaHostAlloc, or any pinned
 * allocation under UVA); the plan's kernels then read inputs and write
 * outputs over PCIe directly, the transfer fused with the stitched compute.
 * Fails (status != 0, nothing launched) for pageable buffers. */
int stc_exec_run_host_zero_copy(stc_exec* e, const void* const* inputs, void* const* outputs);
/* In-graph kernel timeline of one replay (diagnostics; the exec must have been
 * created with STITCH_TRACE=1 in the environment): start_us[i] / end_us[i] =
 * first CTA entry / last CTA exit of kernel i (%globaltimer), us since the
 * earliest entry; -1 for library (GEMM) units.  Arrays of num_kernels
 * entries -- for a plan run by the persistent template ("persistent(U)", one
 * kernel) 1 + U: entry 1+u = unit u ready (producers counted) / done; for the
 * resident template ("resident(U units, S steps, cluster C)", one kernel)
 * 1 + S: entry 1+s = step s (first CTA entering / last CTA leaving).  With
 * STITCH_TRACE_CTAS=c as well, every entry k is recorded per CTA b < c at
 * index k*c + b (arrays c times longer). */
int stc_exec_trace(stc_exec* e, double* start_us, double* end_us);
/* Pipelined host execution over chunks of DIFFERENT sizes: chunk k runs on
 * execs[exec_of_chunk[k]] (each exec built from a shard graph of the same
 * graph, e.g. batch 1 / 3 / 4); chunk k of a chunked input starts right after
 * chunk k-1's bytes.  Small first/last chunks shorten the pipeline's fill and
 * drain.  Same result as running the chunks one by one. */
int stc_exec_run_host_pipeline(stc_exec* const* execs, const int* exec_of_chunk, int nchunks,
                               const void* const* inputs, void* const* outputs, const int* input_chunked);
int stc_exec_upload(stc_exec* e, const void* const* inputs);
/* async graph replay on `cuda_stream` using buffer set `set` (0 = the
 * uploaded buffers; see stc_exec_prepare_sets).  NULL selects the executor's
 * own non-blocking stream -- NOT the legacy default stream -- so a caller that
 * times with events must pass the stream it records them on. */
int stc_exec_launch(stc_exec* e, void* cuda_stream, int set);
/* allocate `sets` independent copies of every buffer and copy set 0's
 * parameters into them, so timed replays can rotate through more bytes than
 * L2 holds with HBM-resident (cold) inputs */
int stc_exec_prepare_sets(stc_exec* e, int sets);
int stc_exec_download(stc_exec* e, void* const* outputs);
int stc_exec_sync(stc_exec* e);
/* device buffer of a graph tensor (parameter/output/kernel boundary) */
int stc_exec_tensor(const stc_exec* e, const char* name, void** dptr, size_t* bytes);
/* Timing with CUDA events on the exec stream.  sets >= 1 independent copies
 * of every buffer are rotated between replays so the working set exceeds L2
 * (sets*bytes > L2) - inputs stay HBM-resident but cold.  Outputs:
 * us_per_run = average graph replay time; kernel_us[i] (optional, length
 * num_kernels) = average duration of kernel i measured by per-kernel events. */
int stc_exec_time(stc_exec* e, int iters, int warmup, int sets, double* us_per_run,
                  double* kernel_us);
/* Latency of ONE call on the device: each replay (set rotated as above) is
 * queued behind a warp spinning on the global timer, so the events around it
 * bracket the replay's device time -- launch-to-completion of an idle device
 * -- and not the host's submission of the launch.  us_per_call = average
 * over iters; kernel_us[i] (optional) = kernel i launched on its own between
 * events (same spin prelude).  No equivalent in the reference (it has no
 * device path); the figure behind the bench's single-call roofline. */
int stc_exec_time_call(stc_exec* e, int iters, int warmup, int sets, double* us_per_call,
                       double* kernel_us);
/* Batched replay: `steps_per_graph` consecutive steps (rotating buffer sets)
 * captured into ONE CUDA Graph so the graph-launch cost is paid once per
 * batch (the paper's launch-overhead argument applied across batches).
 * prepare -> *n_graphs batch graphs; launch_batch replays graph `index`. */
int stc_exec_prepare_batches(stc_exec* e, int sets, int steps_per_graph, int* n_graphs);
int stc_exec_launch_batch(stc_exec* e, void* cuda_stream, int index);
int stc_exec_time_batched(stc_exec* e, int steps, int warmup, int sets, int steps_per_graph,
                          double* us_per_step);

/* ---- low-level runtime (the CUDA layer the executor is built on) --------- */
/* NVRTC -arch=sm_100a compile with the on-disk cubin cache; returns the
 * cache key (hex) of the cubin so callers can reuse it */
int stc_compile(const char* cuda_source, const char* options, char** cubin_key);
/* directory of the cubin cache ($STITCH_CACHE_DIR or <pkg>/lib/cubin_cache) */
const char* stc_cache_dir(void);

/* Device context, modules, ctx-owned buffers and explicit CUDA Graphs
 * (stc_init / stc_compile(ctx, ...) / stc_alloc / stc_free /
 * stc_upload / stc_download / stc_graph_* / stc_nccl_gather; renamed
 * stc_ctx_* / stc_cgraph_* because stc_graph_* and stc_free already name the
 * IR graph and the string deallocator).  Lifetime: the ctx owns its buffers;
 * modules and graphs are destroyed by their own *_destroy.  One ctx per GPU,
 * driven by one host thread. */
typedef struct stc_ctx stc_ctx;
typedef struct stc_module stc_module;
typedef struct stc_cgraph stc_cgraph;
typedef struct stc_comm stc_comm;
int stc_ctx_create(int device, stc_ctx** out);
void stc_ctx_destroy(stc_ctx* c);
/* NVRTC sm_100a (cached); every named kernel is resolved now */
int stc_ctx_compile(stc_ctx* c, const char* cuda_source, const char* const* kernel_names, int n,
                    stc_module** out);
void stc_module_destroy(stc_module* m);
int stc_ctx_alloc(stc_ctx* c, size_t bytes, void** dptr);
int stc_ctx_release(stc_ctx* c, void* dptr);
int stc_ctx_upload(stc_ctx* c, void* dptr, const void* host, size_t bytes);
int stc_ctx_download(stc_ctx* c, void* host, const void* dptr, size_t bytes);
/* kernels added in order run in order (each depends on the previous);
 * args = array of pointers to the argument values, as cudaLaunchKernel */
int stc_cgraph_create(stc_ctx* c, stc_cgraph** out);
int stc_cgraph_add_kernel(stc_cgraph* g, stc_module* m, const char* name, int grid, int block, int smem_bytes,
                          int cooperative, void** args);
int stc_cgraph_instantiate(stc_cgraph* g);
int stc_cgraph_launch(stc_cgraph* g, void* cuda_stream);
/* average CUDA-event time of one replay over `iters`, L2 flushed before each
 * replay when flush_bytes > 0 (a buffer that large is written) */
int stc_cgraph_time(stc_cgraph* g, int iters, size_t flush_bytes, float* us_per_iter);
void stc_cgraph_destroy(stc_cgraph* g);
/* NCCL (libnccl.so.2 loaded on first use) for the verification gather of
 * shard outputs -- never on the timed data path.  The 128-byte unique id is
 * created on one rank and shared out of band. */
int stc_nccl_unique_id(char* id128);
int stc_nccl_comm_init(stc_ctx* c, int nranks, int rank, const char* id128, stc_comm** out);
int stc_nccl_gather(stc_comm* cm, const void* send, void* recv, size_t bytes_per_rank, void* cuda_stream);
void stc_nccl_comm_destroy(stc_comm* cm);

/* ---- drop-in pipeline ------------------------------------------------------
 * replaces stitch::run_pipeline (include/stitch/pipeline.hpp:28): writes
 * plan.json, kernels/kNNN_<producer>.stitch, report.txt, [graph.dot];
 * run_sim executes the plan on the GPU and compares with the unfused
 * execution (rel 1e-4, abs 1e-5).  Returns 0 / 1 / 2 like the reference. */
int stc_run_pipeline(const char* graph_path, const char* device_config_path, int k,
                     int beam_width, const char* output_dir, int emit_dot, int run_sim,
                     int run_baseline, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif /* STITCH_B200_H */
