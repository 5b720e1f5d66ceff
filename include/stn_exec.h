/*
 * stn_exec.h -- C ABI of the B200-native stem executor (sm_100a).
 *
 * This is the drop-in boundary for the per-slice hot path of the reference
 * `stemtn` runtime (/root/reference/proj/include/stemtn/runtime.hpp). The
 * reference keeps building the tensor network, planning the contraction and
 * lowering it with `compile()` (runtime.hpp:243-358); the lowered
 * `ExecutablePlan` (runtime.hpp:60-73) is flattened into the plain-old-data
 * `stn_plan_desc` below and every executor entry point of runtime.hpp maps to
 * one function here:
 *
 *   reference (runtime.hpp)                         this ABI
 *   ----------------------------------------------  -----------------------------
 *   ExecutablePlan (60-73), from compile (243)      stn_plan_create / stn_plan_destroy
 *   plan.net vertex tensors poked by the sampler     stn_plan_set_leaf_values
 *     (sampler.hpp:206-213)
 *   build_branch_cache (492-500)                    stn_cache_build / stn_cache_destroy
 *   BranchCache fields (146-152)                    stn_cache_info
 *   run_subtask (502-514) -> SubtaskResult (75-81)  stn_run_subtask
 *   run_subtask on an explicit digit vector          stn_run_subtask_digits
 *     (assignment decode at runtime.hpp:371-378,
 *      for plans whose uint64 subtasks() overflows,
 *      scheme.hpp:33-37)
 *   worker envelope [lo,hi) (queue.hpp:250-252)     stn_run_slices
 *   run_scheme (555-632) -> (Tensor, RunReport)     stn_run_scheme
 *   stemtn::Error / ErrorKind (errors.hpp:8-74)     stn_status + stn_last_error
 *
 * Conventions: every function returns an stn_status; on failure a message is
 * available from stn_last_error() (thread-local). Complex values are
 * interleaved (re, im) pairs. Output tensors use the reference's layout: axes
 * are the root's alive edges (the open edges) in ascending edge-id order,
 * row-major (runtime.hpp:341-346, 417). `stream` arguments are cudaStream_t
 * passed as void*; NULL means the legacy default stream.
 */
#ifndef STN_EXEC_H_
#define STN_EXEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define STN_ABI_VERSION 1

/* Status codes. 1..19 mirror stemtn::ErrorKind (errors.hpp:8-30) as
 * (enumerator index + 1); >= 100 are executor-side conditions. */
typedef enum stn_status {
  STN_OK = 0,
  STN_ERR_MALFORMED_NETWORK = 1,
  STN_ERR_CAP_EXCEEDED = 2,
  STN_ERR_OPEN_EDGE_SLICED = 3,
  STN_ERR_INDEX_OUT_OF_RANGE = 4,
  STN_ERR_MISSING_PARAMS = 5,
  STN_ERR_SYNTAX_ERROR = 6,
  STN_ERR_INVARIANT_VIOLATION = 7,
  STN_ERR_QUBIT_COVERAGE = 8,
  STN_ERR_LAYOUT_TOO_SMALL = 9,
  STN_ERR_INFEASIBLE = 10,
  STN_ERR_EDGE_NOT_FOUND = 11,
  STN_ERR_SCHEMA_ERROR = 12,
  STN_ERR_STUCK = 13,
  STN_ERR_HASH_MISMATCH = 14,
  STN_ERR_WIDTH_EXCEEDS_BUDGET = 15,
  STN_ERR_SUBTASK_FAILURE = 16,
  STN_ERR_MISSING_RESULT = 17,
  STN_ERR_CHECKSUM_MISMATCH = 18,
  STN_ERR_EMPTY_SAMPLES = 19,
  STN_ERR_CUDA = 100,             /* a CUDA runtime/driver call failed */
  STN_ERR_INVALID_ARGUMENT = 101, /* NULL pointer, bad size, bad enum */
  STN_ERR_OUT_OF_MEMORY = 102,    /* device arena does not fit */
  STN_ERR_NO_DEVICE = 103,        /* no CUDA device / not sm_100 */
  STN_ERR_IO = 104                /* plan file read/write failed */
} stn_status;

/* Precision of the executed arithmetic (runtime.hpp:23). */
typedef enum stn_precision { STN_SINGLE = 0, STN_DOUBLE = 1 } stn_precision;

/* Kernel policy. EXACT runs every step on SIMT kernels that reproduce the
 * reference loop order and IEEE rounding (no FMA contraction), so results are
 * bitwise identical to the reference CPU path in both precisions. FAST (the
 * default) sends compute-bound single-precision steps to the tcgen05 split-TF32
 * complex GEMM and lets SIMT kernels contract into FMAs; results then agree
 * with the reference within the tolerance stated in DESIGN.md. */
typedef enum stn_mode { STN_MODE_FAST = 0, STN_MODE_EXACT = 1 } stn_mode;

/* One lowered pairwise contraction: a flattened stemtn::Step (runtime.hpp:41-49)
 * plus the D/M/K/N axis-group sizes that compile() derives (runtime.hpp:306-319).
 * Operand/produced axis orders:
 *   lhs  [D|M|K] = lhs canonical axes permuted by lperm   (lrank = nd+nm+nk)
 *   rhs  [D|K|N] = rhs canonical axes permuted by rperm   (rrank = nd+nk+nn)
 *   out  canonical axis i = produced [D|M|N] axis operm[i] (orank = nd+nm+nn)
 * "Canonical" means axes sorted by ascending edge id (the reference's layout). */
typedef struct stn_step_desc {
  int32_t node, lhs, rhs; /* exec-tree node ids */
  int32_t is_branch;      /* 1 = slice-invariant (runtime.hpp:347) */
  int32_t nd, nm, nk, nn; /* number of D/M/K/N axes */
  int64_t D, M, N, K;     /* products of the group dims */
  uint64_t mults;         /* D*M*N*K */
  int32_t lrank, rrank, orank;
  const int32_t *lperm;    /* [lrank] */
  const int32_t *rperm;    /* [rrank] */
  const int32_t *operm;    /* [orank] */
  const int32_t *out_dims; /* [orank], canonical output dims */
} stn_step_desc;

/* One leaf of the executed tree: a flattened stemtn::LeafPrep (runtime.hpp:51-58)
 * together with the vertex tensor it loads (network.hpp Vertex). */
typedef struct stn_leaf_desc {
  int32_t node, vertex;
  int32_t rank;          /* original tensor rank */
  const int32_t *dims;   /* [rank] original tensor dims */
  const double *values;  /* [2*prod(dims)] interleaved complex, row-major */
  int32_t n_sliced;      /* number of restricted axes */
  const int32_t *sliced_axis;  /* [n_sliced] axis in the original tensor, descending */
  const int32_t *sliced_index; /* [n_sliced] index into the plan's sliced-edge list */
  int32_t perm_rank;     /* rank after restriction */
  const int32_t *perm;   /* [perm_rank] post-restriction axes -> ascending edge id */
} stn_leaf_desc;

/* A flattened stemtn::ExecutablePlan. */
typedef struct stn_plan_desc {
  int32_t precision;      /* stn_precision (CompileOptions.precision) */
  int32_t merge_min_dim;  /* CompileOptions.merge_min_dim */
  int32_t n_nodes;        /* exec_tree node count (2n-1) */
  int32_t root;           /* exec_tree root node id */
  uint64_t identity;      /* plan.identity (runtime.hpp:351-356) */
  uint64_t subtasks;      /* plan.subtasks; 0 when the uint64 product overflowed */
  int32_t merged_groups;
  int32_t exec_cw;
  int32_t n_sliced;             /* |sliced_edges| */
  const int32_t *sliced_dims;   /* [n_sliced], in ascending sliced-edge-id order */
  int32_t n_open;               /* number of open edges (root rank for circuits) */
  int32_t n_steps;
  const stn_step_desc *steps;   /* post-order over exec_tree internals */
  int32_t n_leaves;
  const stn_leaf_desc *leaves;
} stn_plan_desc;

typedef struct stn_plan stn_plan;   /* device-resident plan (opaque) */
typedef struct stn_cache stn_cache; /* device-resident branch cache (opaque) */

/* Per-subtask bookkeeping, the non-tensor fields of SubtaskResult (runtime.hpp:75-81). */
typedef struct stn_subtask_info {
  uint64_t assignment;
  int32_t step_count;
  uint64_t mults;
  uint64_t peak_elements;
} stn_subtask_info;

/* RunReport fields (runtime.hpp:516-541) that the executor fills. Planner-side
 * costs (log2_tc, cw) stay with the caller, which owns the ContractionScheme. */
typedef struct stn_run_report {
  uint64_t subtasks;
  uint64_t mult_count;
  uint64_t branch_mults;
  double wall_seconds;
  double p50_ms, p90_ms, p99_ms; /* per-slice device time */
  int32_t parallelism;
  int32_t precision;
  uint64_t peak_elements;
  int32_t merged_groups;
  int32_t slices_per_batch;       /* slices executed per batched pass */
  int32_t kernel_launches;        /* executor kernels launched by the call */
} stn_run_report;

/* Static plan facts for the caller (shapes, arena size, kernel choice). */
typedef struct stn_plan_info {
  uint64_t identity;
  uint64_t subtasks;
  int32_t n_sliced;
  int32_t out_rank;
  int64_t out_elements;          /* elements of the root tensor */
  int32_t out_dims[64];          /* first out_rank entries valid */
  int32_t per_slice_steps;       /* steps executed per slice when a cache is used */
  uint64_t per_slice_mults;
  uint64_t branch_mults;
  uint64_t peak_elements;        /* largest per-slice intermediate */
  uint64_t arena_bytes_per_slice;
  uint64_t cache_bytes;
  int32_t steps_tensor_core;     /* per-slice steps on the tcgen05 GEMM */
  int32_t steps_absorb;          /* per-slice steps on the bandwidth absorb kernel */
  int32_t steps_generic;         /* per-slice steps on the generic SIMT kernel */
  int32_t sweeps;                /* fused stem sweeps in the per-slice program */
  int32_t steps_in_sweeps;       /* per-slice steps executed inside sweeps */
} stn_plan_info;

/* Per-kernel-class timing of the launches made while profiling is on (CUDA
 * events around every launch, on the launch stream). `bytes` and `flops` are
 * ALGORITHMIC: operand reads + result writes of the contraction (slice-
 * invariant operands counted once per batch) and 8 real flops per complex
 * multiply-add (runtime.hpp:330 `mults`). */
typedef enum stn_kernel_kind {
  STN_KERNEL_GENERIC = 0,   /* strided SIMT contraction (any dims, D batches) */
  STN_KERNEL_ABSORB = 1,    /* bond-2 bandwidth absorb (big stem x small branch) */
  STN_KERNEL_GEMM_SIMT = 2, /* tiled SIMT complex GEMM */
  STN_KERNEL_GEMM_TC = 3,   /* tcgen05 split-TF32 complex GEMM */
  STN_KERNEL_PERMUTE = 4,   /* operand/result axis permutation */
  STN_KERNEL_LEAF = 5,      /* per-slice leaf gather */
  STN_KERNEL_ROOT = 6,      /* ordered fp64 root accumulation */
  STN_KERNEL_ABSORB_TC = 7, /* tcgen05 split-TF32 absorb (K x N >= 64) */
  STN_KERNEL_SWEEP = 8,     /* fused chain of stem absorbs (one HBM pass) */
  STN_KERNEL_KINDS = 9
} stn_kernel_kind;

typedef struct stn_kernel_profile {
  int32_t kind;     /* stn_kernel_kind */
  int32_t launches;
  double ms;        /* summed device time of the launches */
  double bytes;     /* summed algorithmic bytes */
  double flops;     /* summed algorithmic flops */
} stn_kernel_profile;

/* Per-step accumulation of the same timings (one entry per plan step that ran
 * while profiling was on): which kernel took the step and what it cost. */
typedef struct stn_step_profile {
  int32_t step;     /* index into stn_plan_desc.steps */
  int32_t kind;     /* stn_kernel_kind of the step's main kernel */
  int64_t M, N, K;
  int32_t launches; /* all launches of the step (incl. permutes / pre-passes) */
  double ms, bytes, flops;
} stn_step_profile;

/* ---- library ---------------------------------------------------------------- */
const char *stn_version(void);
int stn_abi_version(void);
const char *stn_last_error(void);
const char *stn_status_name(int status);

/* ---- plan files (host only; no device needed) --------------------------------
 * A plan file is the serialized stn_plan_desc (little-endian, "STNPLAN1"). The
 * descriptor returned by stn_plan_load owns its arrays; free it with
 * stn_plan_desc_free. */
int stn_plan_load(const char *path, stn_plan_desc **out);
int stn_plan_save(const stn_plan_desc *desc, const char *path);
void stn_plan_desc_free(stn_plan_desc *desc);

/* ---- device plan -------------------------------------------------------------- */
/* Validates the descriptor, derives per-step contraction geometry, chooses a
 * kernel per step, plans the liveness arena and uploads the leaf tensors to
 * `device`. `mode` is an stn_mode. */
int stn_plan_create(const stn_plan_desc *desc, int device, int mode, stn_plan **out);
int stn_plan_destroy(stn_plan *plan);
int stn_plan_get_info(const stn_plan *plan, stn_plan_info *info);
/* Replaces the tensor of network vertex `vertex` (n_complex interleaved pairs).
 * Existing branch caches become stale: running them fails with
 * STN_ERR_SUBTASK_FAILURE, as a cache of a different plan does in the reference
 * (runtime.hpp:505-507). */
int stn_plan_set_leaf_values(stn_plan *plan, int32_t vertex, const double *values,
                             int64_t n_complex);
/* Upper bound on slices executed together in one batched pass (0 = automatic). */
int stn_plan_set_max_batch(stn_plan *plan, int32_t max_batch);
/* Streams ("lanes", each with its own arena) that stn_run_slices* rotate batches of
 * slices over (default 1; bounded by free device memory). Results are bitwise the
 * same for any value: roots are folded in ascending slice order through an event
 * chain. stn_run_scheme uses its `parallelism` argument instead. */
int stn_plan_set_streams(stn_plan *plan, int32_t streams);

/* Turns per-launch event timing on/off (off by default) and reads the totals
 * accumulated since the last reset; out must hold STN_KERNEL_KINDS entries.
 * Reading synchronizes on the recorded events. */
int stn_plan_set_profiling(stn_plan *plan, int enable);
int stn_plan_get_profile(stn_plan *plan, stn_kernel_profile *out);
int stn_plan_reset_profile(stn_plan *plan);
/* Copies up to `cap` per-step entries (steps with at least one timed launch, in
 * plan order) into out; *n receives the number of such steps. */
int stn_plan_get_step_profile(stn_plan *plan, stn_step_profile *out, int32_t cap, int32_t *n);

/* ---- branch cache ------------------------------------------------------------ */
int stn_cache_build(stn_plan *plan, void *stream, stn_cache **out);
int stn_cache_destroy(stn_cache *cache);
int stn_cache_info(const stn_cache *cache, uint64_t *plan_identity, uint64_t *mults,
                   uint64_t *elements);

/* ---- execution ------------------------------------------------------------- */
/* One subtask. `out_host` receives 2*out_elements doubles (the root tensor
 * converted to double, as to_tensor does at runtime.hpp:103-110). `cache` may be
 * NULL (every step, branch ones included, runs for this assignment). `info` may
 * be NULL. Blocks until the result is on the host. */
int stn_run_subtask(stn_plan *plan, uint64_t assignment, const stn_cache *cache, void *stream,
                    double *out_host, stn_subtask_info *info);
/* Same, with the sliced-edge digits given explicitly (digits[i] in
 * [0, sliced_dims[i])); `info->assignment` is set to 0. */
int stn_run_subtask_digits(stn_plan *plan, const int32_t *digits, const stn_cache *cache,
                           void *stream, double *out_host, stn_subtask_info *info);
/* Slices [lo, hi) with a branch cache. Asynchronous on `stream`. If `acc_dev`
 * is not NULL, the per-slice roots are converted to double and added to it
 * (2*out_elements doubles, device memory) in ascending assignment order. If
 * `per_slice_dev` is not NULL, slice a's root (as doubles) is stored at
 * per_slice_dev + (a - lo) * 2 * out_elements. */
int stn_run_slices(stn_plan *plan, const stn_cache *cache, uint64_t lo, uint64_t hi, void *stream,
                   double *acc_dev, double *per_slice_dev);
/* Same as stn_run_slices for an explicit list of digit vectors
 * (n_slices x n_sliced, row-major host memory). */
int stn_run_slices_digits(stn_plan *plan, const stn_cache *cache, const int32_t *digits,
                          uint64_t n_slices, void *stream, double *acc_dev,
                          double *per_slice_dev);
/* Whole scheme on one device: builds the branch cache, runs every subtask and
 * sums the results in ascending assignment order in double, so the output is
 * bit-stable for any `parallelism` (runtime.hpp:552-605). `out_host` receives
 * 2*out_elements doubles; `report` may be NULL. */
int stn_run_scheme(stn_plan *plan, int parallelism, double *out_host, stn_run_report *report);

/* Sums `n_slices` per-slice results stored as in stn_run_slices' per_slice_dev
 * into out_dev in ascending order (device, asynchronous). Used after a
 * cross-GPU exchange to reproduce run_scheme's reduction order exactly. */
int stn_sum_slices_ordered(const double *per_slice_dev, uint64_t n_slices, int64_t out_elements,
                           double *out_dev, void *stream);

/* Continues an ascending-order fold: acc_dev[i] = (((acc_dev[i] + r_0[i]) + r_1[i]) + ...)
 * over `n_slices` per-slice rows (device, asynchronous). A fold that starts from
 * zeros on the device owning the first slices and continues on the next device
 * with the accumulator it hands over reproduces run_scheme's sequential sum
 * (runtime.hpp:601-605) bit for bit across any number of GPUs. */
int stn_fold_slices_ordered(const double *per_slice_dev, uint64_t n_slices, int64_t out_elements,
                            double *acc_dev, void *stream);

/* A worker envelope with HOST buffers (queue.hpp:250-252: run_subtask for every
 * assignment of [lo, hi) and hand the results back): slices are the assignments
 * [lo, lo + n_slices) when `digits` is NULL, else the n_slices digit vectors in
 * `digits` (n_slices x n_sliced, row-major). `per_slice_host` (n_slices x
 * 2*out_elements doubles) and `sum_host` (2*out_elements, ascending fold from
 * zero) may each be NULL. Blocks until the results are on the host. */
int stn_run_slices_host(stn_plan *plan, const stn_cache *cache, const int32_t *digits,
                        uint64_t lo, uint64_t n_slices, void *stream, double *per_slice_host,
                        double *sum_host);

/* Frees the process-wide cache of large device blocks that destroyed plans and
 * caches leave behind for reuse (arenas, workspaces >= 64 MiB; STN_BLOCK_CACHE=0
 * disables the cache). */
int stn_flush_block_cache(void);

/* ---- several GPUs of one box -------------------------------------------------
 * The reference's multi-worker layer (queue.hpp:197-336: envelopes of slices
 * claimed by workers, summed by agent_collect in ascending order) and the
 * threads of run_scheme (runtime.hpp:564-598), on the GPUs of one box: one
 * device plan + HBM-resident branch cache per GPU, one host thread per GPU, each
 * GPU a contiguous balanced shard of the slices. Two reductions:
 *   deterministic = 1  every GPU keeps its per-slice roots; the ascending fold
 *                      starts on the first GPU and continues on the next with the
 *                      handed-over 2*out_elements accumulator (a peer copy over
 *                      NVLink per hop): bitwise equal to run_scheme for any
 *                      device count.
 *   deterministic = 0  every GPU folds its own shard; one NCCL all-reduce
 *                      (ncclFloat64, ncclSum) over NVLink combines the partial
 *                      amplitudes (NCCL is loaded at run time with dlopen).
 * `devices` may be NULL (devices 0..n_devices-1). */
typedef struct stn_multi stn_multi;
/* Number of CUDA devices visible to this process (0 without a GPU). */
int stn_device_count(void);
int stn_multi_create(const stn_plan_desc *desc, int n_devices, const int32_t *devices, int mode,
                     stn_multi **out);
int stn_multi_destroy(stn_multi *m);
int stn_multi_device_count(const stn_multi *m);
/* The device plan of GPU i (owned by m), e.g. for stn_plan_get_info / profiling. */
stn_plan *stn_multi_plan(stn_multi *m, int i);
/* Rebuilds every GPU's branch cache (after stn_multi_set_leaf_values). */
int stn_multi_build_caches(stn_multi *m);
int stn_multi_set_leaf_values(stn_multi *m, int32_t vertex, const double *values,
                              int64_t n_complex);
/* run_scheme (runtime.hpp:555-632) over every GPU: all subtasks, summed in
 * ascending assignment order (deterministic = 1) or through one NCCL all-reduce. */
int stn_multi_run_scheme(stn_multi *m, int deterministic, double *out_host,
                         stn_run_report *report);
/* Slices given as assignments [lo, lo + n_slices) (digits NULL) or digit vectors
 * (n_slices x n_sliced host array), sharded over the GPUs; outputs as in
 * stn_run_slices_host. */
int stn_multi_run_slices(stn_multi *m, const int32_t *digits, uint64_t lo, uint64_t n_slices,
                         int deterministic, double *per_slice_host, double *sum_host);
/* One-call form of stn_multi_create + stn_multi_run_scheme + stn_multi_destroy. */
int stn_run_scheme_multi(const stn_plan_desc *desc, int n_devices, const int32_t *devices,
                         int mode, int deterministic, double *out_host, stn_run_report *report);

/* ---- diagnostics --------------------------------------------------------------
 * Runs the tcgen05 split-TF32 complex GEMM on seeded random operands
 * (C = A[M x K] * B[K x N], `batches` independent problems; a_batched /
 * b_batched select per-batch or shared operands) and compares it with an fp64
 * SIMT GEMM of the same inputs. Returns the max |C_tc - C_ref| / max|C_ref| and
 * the mean device time of the tensor-core path (pre-pass + GEMM), of the
 * GEMM kernel alone and of the fp32 SIMT GEMM over `reps` launches, and the
 * fp32 SIMT GEMM's own error for comparison. STN_ERR_INVALID_ARGUMENT if the shape
 * is not supported by the tensor-core kernel. */
int stn_selftest_gemm_tc(int64_t M, int64_t N, int64_t K, int32_t batches, int32_t a_batched,
                         int32_t b_batched, int32_t reps, double *max_rel_err, double *ms_total,
                         double *ms_gemm, double *ms_simt, double *simt_rel_err);

/* Code-generation check (no device needed): emits the NVRTC source of a synthetic
 * fused stem chain (the plan-specialised kernels of chain_jit.cpp) and compiles it
 * for sm_100a; `log` (may be NULL) receives the compiler log. */
int stn_selftest_chain_jit(int exact, char *log, int32_t log_cap);

/* Memory-pipeline check: a 2^log2_elems complex64 tensor is bit-permuted by
 * the tiled absorb kernel (perm[i] = source bit of output bit i; identity when
 * NULL) and copied with cudaMemcpyAsync; returns GB/s (read + write) of both
 * and whether the permutation result is correct. */
int stn_selftest_bitperm(int32_t log2_elems, const int32_t *perm, int32_t reps, double *gbs_kernel,
                         double *gbs_memcpy, int32_t *correct);

#ifdef __cplusplus
}
#endif

#endif /* STN_EXEC_H_ */
