/*
 * amlt_gpu.h — C-ABI of the B200 (sm_100a) backend for AMULET's
 * matrix-multiplication-like task (MMLT):
 *
 *     R[i][j] (+)= sum_k body(A[i][k], B[k][j], per-column vectors[j])
 *
 * This is the drop-in boundary for the reference engine's executor and tuner
 * (reference = /root/reference/proj, "amlt"). Plain C types only: pointers,
 * sizes, enums. No CUDA, C++ or torch types appear in any signature; device
 * buffers are passed as raw device pointers, streams as `void*`.
 *
 * Reference interfaces replaced (file:line in /root/reference/proj):
 *   amlt_gpu_run_subtask       <- run_subtask(plan, kernel, ops, TileParams,
 *                                 Bounds, Clock&, ExecLog*)
 *                                 include/amlt/tiled_executor.hpp:42-44,
 *                                 src/tiled_executor.cpp:9-77
 *   amlt_gpu_adaptive_execute  <- adaptive_execute(plan, kernel, ops, Bounds,
 *                                 pack, Clock&, ExecLog*) -> TuneReport
 *                                 include/amlt/autotuner.hpp:68-70,
 *                                 src/autotuner.cpp:103-151
 *   amlt_gpu_run_host          <- run_fixed / run_adaptive over host-resident
 *                                 MatrixBuffers (src/engine.cpp:165-175)
 *   amlt_gpu_plan_create       <- compile_task(...) -> CompiledTask
 *                                 (src/engine.cpp:86-102): the recognised
 *                                 body, its leaf roles and operand layouts
 *   amlt_body_desc             <- Mmlt + ExprDag identity (recognize.hpp:28-42,
 *                                 expr_dag.hpp:26) reduced to the five bodies
 *   amlt_operands / amlt_matrix<- Operands (kernel_exec.hpp:17-24) over
 *                                 MatrixBuffer (matrix.hpp:14-59)
 *   amlt_bounds                <- Bounds (tiled_executor.hpp:17-21)
 *   amlt_tile_params           <- TileParams (tiled_executor.hpp:11-15)
 *   amlt_exec_record           <- ExecRecord (tiled_executor.hpp:25-34)
 *   amlt_trial / amlt_cover_rect / amlt_tune_report
 *                              <- Trial / CoverRect / TuneReport
 *                                 (autotuner.hpp:11-34)
 *   amlt_clock_fn              <- Clock::now() (clock.hpp:12-16)
 *   amlt_status                <- EngineError hierarchy (errors.hpp:10-60)
 *   amlt_spr                   <- spr (engine.hpp:83-85, src/engine.cpp:212-216)
 *
 * Threading: one caller thread per context. Every call that
 * returns an elapsed time is synchronous; amlt_gpu_enqueue is the
 * asynchronous form (stream-ordered, no clock reads).
 */
#ifndef AMLT_GPU_H
#define AMLT_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMLT_GPU_ABI_VERSION 4

/* Aux arrays one generated (AMLT_BODY_GENERIC) statement may name. */
#define AMLT_MAX_AUX 8

/* Error codes; the C++ shim (amlt_gpu.hpp) rethrows the matching
 * EngineError subclass (errors.hpp:10-60). */
typedef enum {
    AMLT_OK = 0,
    AMLT_ERR_ENGINE = 1,             /* EngineError                          */
    AMLT_ERR_UNSUPPORTED = 2,        /* UnsupportedExpression                */
    AMLT_ERR_MISSING_BINDING = 3,    /* MissingBinding (absent aux operand)  */
    AMLT_ERR_NO_FEASIBLE_KERNEL = 4, /* NoFeasibleKernel                     */
    AMLT_ERR_NON_POSITIVE_TIME = 5,  /* NonPositiveTime                      */
    AMLT_ERR_INVALID_ARGUMENT = 6,   /* bad pointer / bounds / shape         */
    AMLT_ERR_CUDA = 7,               /* CUDA runtime error                   */
    AMLT_ERR_NO_DEVICE = 8           /* no usable sm_100 device              */
} amlt_status;

/* The five BASELINE bodies (+ q3's threshold count):
 *   GEMM      R += A*B                                  preset matmul
 *   DISCOUNT  R += A*B - (A*B > T)*A*B*dis[j]           preset q1
 *   BOOST     R += A*B + (A*B > T)*(A*B - T)            preset q2
 *   SQDIFF    R += (A - B)*(A - B)
 *   EQCOUNT   R += A == B
 *   THRCOUNT  R += A*B > T                              preset q3
 * and GENERIC: any other recognised multiply-accumulate-like statement
 * (recognize.cpp:84-166: one A[i][k]/A[k][i], one B[k][j]/B[j][k], aux
 * leaves that are scalars, [i], [j] or [i][j]; + - * / and comparisons).
 * Its body is generated from the statement and compiled at plan time
 * (NVRTC) into the same tile kernels; such plans come only from
 * amlt_gpu_plan_from_source.                                               */
typedef enum {
    AMLT_BODY_GEMM = 0,
    AMLT_BODY_DISCOUNT = 1,
    AMLT_BODY_BOOST = 2,
    AMLT_BODY_SQDIFF = 3,
    AMLT_BODY_EQCOUNT = 4,
    AMLT_BODY_THRCOUNT = 5,
    AMLT_BODY_GENERIC = 6
} amlt_body;

typedef enum { AMLT_F64 = 0, AMLT_F32 = 1, AMLT_I32 = 2 } amlt_dtype;

/* MatrixBuffer storage order (matrix.hpp:10). */
typedef enum { AMLT_ROW_MAJOR = 0, AMLT_COL_MAJOR = 1 } amlt_order;

/* Statement-side operand layout (recognize.hpp:19): NORMAL is A[i][k] /
 * B[k][j]; TRANSPOSED is A[k][i] / B[j][k]. */
typedef enum { AMLT_LAYOUT_NORMAL = 0, AMLT_LAYOUT_TRANSPOSED = 1 } amlt_layout;

/* Leaf class of the threshold operand (recognize.hpp:14). */
typedef enum {
    AMLT_LEAF_CONSTANT = 0,
    AMLT_LEAF_VEC_I = 1,
    AMLT_LEAF_VEC_J = 2,
    AMLT_LEAF_MAT_IJ = 3
} amlt_leaf_class;

typedef struct {
    int32_t body;        /* amlt_body                                        */
    int32_t dtype;       /* amlt_dtype: storage AND arithmetic type           */
    int32_t accumulate;  /* 1 for "+=", 0 for "=" (last k wins)               */
    int32_t layout_a;    /* amlt_layout                                       */
    int32_t layout_b;    /* amlt_layout                                       */
    int32_t thres_class; /* amlt_leaf_class of T (DISCOUNT/BOOST/THRCOUNT)    */
    double thres_value;  /* T when thres_class == AMLT_LEAF_CONSTANT          */
} amlt_body_desc;

/* A dense matrix in DEVICE memory, described like a MatrixBuffer: (rows,
 * cols) are the buffer's own dimensions, `ld` its leading stride in
 * elements (row-major: >= cols; col-major: >= rows). Vectors are len x 1. */
typedef struct {
    void* data;
    int64_t rows;
    int64_t cols;
    int64_t ld;
    int32_t order; /* amlt_order */
    int32_t dtype; /* amlt_dtype; must equal the plan's dtype                 */
} amlt_matrix;

/* Operands (kernel_exec.hpp:17-24). `thres` and `dis` are the aux leaves the
 * fixed bodies name; a GENERIC plan binds its aux leaves by position in
 * `aux`, in the order amlt_task_info.aux_names lists them (scalars as 1 x 1,
 * [i] / [j] vectors as len x 1, [i][j] as M x N buffers). A body that needs
 * an absent leaf -> MISSING_BINDING. */
typedef struct {
    amlt_matrix a;
    amlt_matrix b;
    amlt_matrix r;
    amlt_matrix thres; /* data == NULL when unbound */
    amlt_matrix dis;   /* data == NULL when unbound */
    int32_t n_aux;     /* GENERIC plans: bound entries of aux */
    amlt_matrix aux[AMLT_MAX_AUX];
} amlt_operands;

/* Half-open index rectangle (tiled_executor.hpp:17-21). */
typedef struct {
    int64_t i0, i1;
    int64_t j0, j1;
    int64_t k0, k1;
} amlt_bounds;

/* TileParams (tiled_executor.hpp:11-15) on the GPU:
 *   kc      K-segment depth. kc <= 0 or kc >= K: one pass over K. Otherwise
 *           kc is rounded up to a multiple of 16 and the K range is cut
 *           into ceil(K/kc) segments computed in parallel (split-K) and added
 *           to R in ascending segment order (deterministic), the GPU form of
 *           the reference's kc loop.
 *   nc      column-tile width: picks the registered tile variant whose CTA
 *           width is the largest <= nc (nc <= 0: planner default).
 *   pack    accepted for interface parity; operands are always staged
 *           through shared memory, so it has no effect (bit-neutral, as the
 *           reference's packing is, acceptance c8).
 *   variant explicit tile-variant index (>= 0) overriding nc; -1 = by nc. */
typedef struct {
    int64_t kc;
    int64_t nc;
    int32_t pack;
    int32_t variant;
} amlt_tile_params;

/* One launch the executor made (ExecRecord, tiled_executor.hpp:25-34). */
typedef struct {
    int32_t variant;
    int32_t splits; /* K segments of this dispatch */
    int64_t i0, i1, j0, j1, k0, k1;
} amlt_exec_record;

/* Caller-owned dispatch log: the library appends while count < capacity and
 * always increments `total`. */
typedef struct {
    amlt_exec_record* records;
    int32_t capacity;
    int32_t count;
    int32_t total;
} amlt_exec_log;

/* Tile-variant description (the GPU analogue of KernelShape + ledger). */
typedef struct {
    int32_t index;
    int32_t body;
    int32_t dtype;
    int32_t block_m;      /* CTA tile rows                                   */
    int32_t block_n;      /* CTA tile columns                                */
    int32_t block_k;      /* K depth per shared-memory stage                 */
    int32_t thread_m;     /* register micro-tile rows per thread             */
    int32_t thread_n;     /* register micro-tile columns per thread          */
    int32_t threads;      /* threads per CTA                                 */
    int32_t stages;       /* cp.async pipeline depth                         */
    int32_t smem_bytes;   /* dynamic shared memory per CTA                   */
    int32_t tensor_core;  /* 1: DMMA (mma.sync f64) tensor-core variant      */
    char name[48];
} amlt_variant_info;

/* Clock seam (clock.hpp:12-16): seconds, monotonic. When given, it is read
 * exactly twice per subtask, immediately around the synchronous GPU work
 * (tiled_executor.cpp:40,75); when NULL, CUDA events on the context stream
 * time the subtask. */
typedef double (*amlt_clock_fn)(void* user);

#define AMLT_MAX_TRIALS 128
#define AMLT_MAX_COVER 64

typedef struct {
    int64_t value;  /* variant index tried                                   */
    int64_t rows;   /* row band the trial computed (its share of the output) */
    double elapsed; /* seconds                                               */
    double score;   /* elapsed / rows, the band's partial last CTA round
                       counted as full (ceil(c)/c, c = CTAs per SM): lower
                       is better                                         */
} amlt_trial;

/* A completed output region (CoverRect, autotuner.hpp:19-24, extended with
 * the row range because the GPU tuner lays candidates on row bands). */
typedef struct {
    int64_t i0, i1;
    int64_t k0, k1;
    int64_t j0, j1;
} amlt_cover_rect;

typedef struct {
    int32_t n_trials;
    amlt_trial trials[AMLT_MAX_TRIALS];
    int32_t best_variant;
    int64_t best_kc;
    int32_t tuned;      /* 0: too small to tune, ran whole with the default */
    int32_t from_cache; /* 1: winner reused from an earlier tuning          */
    int32_t scratch_tuned; /* 1: too small for row-band trials: candidates
                              timed on the whole task against a scratch R
                              (trials rows == M), then the task ran once    */
    int32_t n_cover;
    amlt_cover_rect coverage[AMLT_MAX_COVER]; /* disjoint, union = bounds   */
    double tuning_fraction;                   /* rows of R produced by trial
                                                 bands / M (scratch trials
                                                 produce none: 0)          */
    double total_seconds;                     /* sum over all subtasks,
                                                 scratch trials included   */
    double tuning_seconds;                    /* of which whole-task trials on
                                                 the scratch R (work redone
                                                 for the real R afterwards) */
    int32_t refined;                          /* row-band tuning whose bands
                                                 were shorter than 8 waves: the
                                                 best `refined` candidates ran
                                                 one more 8-wave band each (the
                                                 last `refined` trials), and
                                                 the best of THOSE won; 0:
                                                 the argmin of all trials won */
} amlt_tune_report;

typedef struct amlt_ctx amlt_ctx;
typedef struct amlt_plan amlt_plan;

/* Context flags. DRY_RUN: no device is touched; dispatches are planned,
 * logged and "timed" through the clock seam only (tests of the host logic
 * on machines without a GPU). Results are never produced in this mode. */
#define AMLT_CTX_DRY_RUN 1
/* F64_EMULATION: lets the tuner choose the f64 GEMM that runs on the int8
 * tensor cores (Ozaki-style exact slicing, ~2x the fp64 DMMA rate). Its error
 * is ~1e-14 normwise on BASELINE's data (bound 1e-12) and exact on integer
 * data, but it scales each row of A / column of B by one power of two, so a
 * row mixing magnitudes more than ~2^40 apart loses the small ones: opt-in.
 * Without the flag the variant runs only when named in amlt_tile_params. */
#define AMLT_CTX_F64_EMULATION 2

int amlt_gpu_abi_version(void);

amlt_status amlt_gpu_ctx_create(int device, int flags, amlt_ctx** out);
void amlt_gpu_ctx_destroy(amlt_ctx* ctx);
/* Message of the last failing call on this context (or of ctx creation when
 * ctx == NULL). Never NULL. */
const char* amlt_gpu_last_error(const amlt_ctx* ctx);
/* Launch on the caller's CUDA stream (cudaStream_t as void*); NULL restores
 * the context's own stream. The own stream is a blocking stream: ordered
 * with the legacy default stream (work the caller queued there before a call
 * is complete when the call's kernels start). Callers producing operands on
 * any other stream pass that stream here. */
amlt_status amlt_gpu_set_stream(amlt_ctx* ctx, void* stream);
/* Forget tuning winners cached by amlt_gpu_adaptive_execute. */
void amlt_gpu_clear_tuning_cache(amlt_ctx* ctx);

/* Pseudo-program opcodes (schedule.hpp:11-15, POpcode order). */
enum {
    AMLT_PROG_MOV = 0, AMLT_PROG_ADD, AMLT_PROG_SUB, AMLT_PROG_MUL, AMLT_PROG_DIV,
    AMLT_PROG_GTCMP, AMLT_PROG_GECMP, AMLT_PROG_LTCMP, AMLT_PROG_LECMP, AMLT_PROG_EQCMP,
    AMLT_PROG_MASKSUB, AMLT_PROG_MASKADD, AMLT_PROG_NOPS
};

/* The compile_task boundary (src/engine.cpp:86-102): which GPU body a task
 * text is, and which arrays play A, B, R, the threshold and the discount
 * vector. Names are "" for absent roles. GENERIC statements list their aux
 * leaves (first-use order) with their index classes. */
typedef struct {
    amlt_body_desc desc; /* dtype left 0; the caller chooses it          */
    char a[64];
    char b[64];
    char r[64];
    char thres[64];
    char dis[64];
    int32_t n_aux;
    char aux_names[AMLT_MAX_AUX][64];
    int32_t aux_class[AMLT_MAX_AUX]; /* amlt_leaf_class */
    /* The reference's compiled program for this statement (build_dag +
     * schedule_labelfs: one pseudo-instruction per DAG op node with equal
     * subexpressions shared, plus the final accumulate; expr_dag.cpp:63-245,
     * schedule.cpp:265-273): instructions per opcode (AMLT_PROG_*), their
     * total, and the body-op flops per inner iteration (add / sub / mul / div /
     * compare 1, masksub / maskadd 2, the final add 1, mov 0): SURVEY §8(d)'s
     * measure (B). */
    int32_t prog_counts[AMLT_PROG_NOPS];
    int32_t prog_instrs;
    int32_t prog_flops;
} amlt_task_info;

/* Parses and recognises a task in the reference DSL. UNSUPPORTED for a task
 * that is not multiply-accumulate-like (the reference then runs it on its
 * CPU interpreter); ENGINE for a parse error. Message:
 * amlt_gpu_last_error(NULL). */
amlt_status amlt_gpu_recognize(const char* task_source, amlt_task_info* info);

amlt_status amlt_gpu_plan_create(amlt_ctx* ctx, const amlt_body_desc* desc, amlt_plan** out);
/* amlt_gpu_recognize + amlt_gpu_plan_create in the given dtype; `info`
 * (optional) receives the roles. */
amlt_status amlt_gpu_plan_from_source(amlt_ctx* ctx, const char* task_source, int dtype,
                                      amlt_plan** out, amlt_task_info* info);
/* The CUDA source amlt_gpu_plan_from_source compiles (NVRTC, sm_100a) for a
 * GENERIC statement: the tile-kernel header plus the generated Body. Writes
 * at most buflen bytes (NUL-terminated) and returns the full length, or -1
 * (message in amlt_gpu_last_error(NULL)) for a fixed-body or unrecognised
 * statement. */
int64_t amlt_gpu_generated_source(const char* task_source, int dtype, char* buf, int64_t buflen);
void amlt_gpu_plan_destroy(amlt_plan* plan);
int amlt_gpu_plan_num_variants(const amlt_plan* plan);
amlt_status amlt_gpu_plan_variant(const amlt_plan* plan, int idx, amlt_variant_info* info);
/* Variant the planner uses when no tuning result applies. */
int amlt_gpu_plan_default_variant(const amlt_plan* plan, int64_t M, int64_t N, int64_t K);

/* run_subtask: R(bounds) (+)= body over bounds, synchronously. Returns the
 * elapsed seconds between the two clock reads in *elapsed_s. */
amlt_status amlt_gpu_run_subtask(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                                 const amlt_tile_params* tile, const amlt_bounds* bounds,
                                 amlt_clock_fn clock, void* clock_user, amlt_exec_log* log,
                                 double* elapsed_s);

/* The per-element device executor (GPU counterpart of run_naive,
 * src/naive.cpp:65-117,157-166, and execute_scalar_region,
 * src/kernel_exec.cpp:408-457): one thread per R element walks k ascending,
 * evaluating the statement term node by node (no contraction) and
 * accumulating `R += v` (or `R = v` for assignments). The untiled reference
 * path behind "naive" runs and --verify; synchronous; timed like
 * run_subtask (two clock reads, or CUDA events when clock is NULL). */
amlt_status amlt_gpu_run_naive(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                               const amlt_bounds* bounds, amlt_clock_fn clock, void* clock_user,
                               double* elapsed_s);

/* Asynchronous form of run_subtask: enqueues on the context stream and
 * returns; no clock reads, no synchronisation. */
amlt_status amlt_gpu_enqueue(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                             const amlt_tile_params* tile, const amlt_bounds* bounds);

/* One enqueue of (plan, ops, tile, bounds) captured into a CUDA graph on the
 * context's stream, for repeated identical steps (launch-bound small tasks:
 * the graph replays every kernel of the step, preparation and split-K
 * reduction included, with no per-launch host work). The operand pointers,
 * shapes and the chosen variant are fixed at capture; amlt_gpu_graph_launch
 * enqueues a replay on the context's current stream and fails with
 * AMLT_ERR_INVALID_ARGUMENT if the context's workspaces were reallocated
 * since the capture (capture again then). */
typedef struct amlt_graph amlt_graph;
amlt_status amlt_gpu_graph_capture(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                                   const amlt_tile_params* tile, const amlt_bounds* bounds,
                                   amlt_graph** out);
amlt_status amlt_gpu_graph_launch(amlt_graph* graph);
void amlt_gpu_graph_destroy(amlt_graph* graph);

/* adaptive_execute: measured choice of the tile variant on row bands of the
 * real task (each band contributes its rows of R; coverage exactly once),
 * then the remainder with the winner. */
amlt_status amlt_gpu_adaptive_execute(amlt_ctx* ctx, const amlt_plan* plan,
                                      const amlt_operands* ops, const amlt_bounds* bounds,
                                      int pack, amlt_clock_fn clock, void* clock_user,
                                      amlt_exec_log* log, amlt_tune_report* report);

/* run_host flags */
#define AMLT_HOST_R_ZERO 1 /* R starts at zero: device R is zero-filled, not copied in */
/* With a communicator attached (amlt_gpu_comm_attach, or a rank of an
 * amlt_sharded group): B and the operands every rank shares (thresholds and
 * leaves indexed by nothing or by j) are read from host memory on rank 0 only
 * and broadcast to the other ranks over NVLink / NVSwitch (NCCL), panel by
 * panel as they land, overlapping compute. Other ranks pass the shapes of
 * those operands with data == NULL; every rank passes its own A / R rows. */
#define AMLT_HOST_BCAST_SHARED 2

/* AMULET's own tuner contract, restated on the GPU executor
 * (src/autotuner.cpp:8-151): find_kc lays kc candidates (K, then repeated
 * ceil-halving down to 16) along K on two i_w-wide column strips and scores
 * elapsed / kc; find_nc scores column strips of width i_w, 2 i_w, ... by
 * elapsed / nc until the first increase or the column budget; the remainder
 * runs with the winners; tasks with N < 4 i_w or fewer than i_h rows run
 * untuned (kc = min(K, 256), nc = N). Every subtask writes R and the (k, j)
 * coverage ledger tiles K x N exactly once. On the GPU, a subtask's kc is its
 * K-segment depth (split-K, ordered reduction) and nc picks the tile width.
 * Pass the reference plan's kernel shape (i_h, i_w) to reproduce its
 * decisions exactly under the same clock script. */
#define AMLT_MAX_REF_TRIALS 64
#define AMLT_MAX_REF_COVER 128

typedef struct {
    int64_t value;  /* kc or nc tried */
    double elapsed;
    double score;   /* elapsed / value */
} amlt_ref_trial;

typedef struct {
    int64_t k0, k1;
    int64_t j0, j1;
} amlt_ref_cover; /* CoverRect: full M rows */

typedef struct {
    int32_t n_kc_trials;
    amlt_ref_trial kc_trials[AMLT_MAX_REF_TRIALS];
    int32_t n_nc_trials;
    amlt_ref_trial nc_trials[AMLT_MAX_REF_TRIALS];
    int64_t best_kc;
    int64_t best_nc;
    int32_t tuned;
    int32_t n_cover;
    amlt_ref_cover coverage[AMLT_MAX_REF_COVER];
    double tuning_fraction;
    double total_seconds;
} amlt_amulet_report;

amlt_status amlt_gpu_adaptive_execute_amulet(amlt_ctx* ctx, const amlt_plan* plan,
                                             const amlt_operands* ops, const amlt_bounds* bounds,
                                             int i_h, int i_w, amlt_clock_fn clock,
                                             void* clock_user, amlt_exec_log* log,
                                             amlt_amulet_report* report);

/* Host-buffer entry (the reference's callers hold host MatrixBuffers:
 * run_fixed / run_adaptive, src/engine.cpp:165-175): operands' `data` are
 * HOST pointers (pinned for full copy bandwidth). A copy / compute pipeline:
 * B in K panels and A in row bands go H2D on a copy stream; the first row
 * band is computed panel by panel as B lands (band 0's A arrives with each
 * panel), its R zero-filled (AMLT_HOST_R_ZERO) or copied in on the device and
 * copied back D2H when done. The other rows:
 *  - R in pinned, device-mapped host memory (cudaHostAlloc / cudaHostRegister)
 *    and a winner whose epilogue allows it: launches whose epilogue writes R
 *    straight into the host buffer (zero-copy; prior values read from there
 *    unless AMLT_HOST_R_ZERO), one launch for all these rows unless the A
 *    copies dominate (then a few row bands). R outside the bounds is never
 *    touched.
 *  - otherwise: whole-K row bands, each R band D2H on a second copy stream as
 *    soon as it is done (R bands zero-filled or copied in like band 0).
 * B is cut into K panels when its k rows are contiguous (B[k][j] row-major,
 * B[j][k] col-major), the winner is not split-K and the statement
 * accumulates. The tile: `tile` if given, else the winner cached by an
 * earlier tuning of the same shape, else the planner default. *elapsed_s
 * covers all copies and compute (the clock, if any, is read exactly twice
 * around all of it). amlt_gpu_last_host_layout reports the layout used. */
amlt_status amlt_gpu_run_host(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* host_ops,
                              const amlt_tile_params* tile, const amlt_bounds* bounds, int flags,
                              amlt_clock_fn clock, void* clock_user, double* elapsed_s);
/* run_adaptive over host buffers: amlt_gpu_run_host whose tile comes from
 * the runtime tuner. When no winner is cached for the shape, the operands
 * are copied whole and the task runs through amlt_gpu_adaptive_execute
 * (row-band or scratch trials, the remainder with the winner; a caller clock
 * scores the trials, read twice around each of them); later calls of the
 * shape reuse the winner through the pipeline. *report: the trials (empty
 * when the winner was cached: from_cache = 1), the winner, and coverage
 * rectangles that are disjoint with union = bounds. */
amlt_status amlt_gpu_run_host_adaptive(amlt_ctx* ctx, const amlt_plan* plan,
                                       const amlt_operands* host_ops, const amlt_bounds* bounds,
                                       int flags, amlt_clock_fn clock, void* clock_user,
                                       amlt_tune_report* report, double* elapsed_s);

/* Multi-process (one process per GPU, e.g. torchrun) communicator for
 * AMLT_HOST_BCAST_SHARED: rank 0 makes an id (AMLT_NCCL_ID_BYTES opaque
 * bytes), the caller hands it to every rank by its own means, and every rank
 * attaches it to its context (collective: blocks until all ranks attach).
 * One rank is valid: the broadcasts are then no-ops (the path is the same).
 * NCCL (libnccl.so.2) is loaded at run time. */
#define AMLT_NCCL_ID_BYTES 128
amlt_status amlt_gpu_comm_unique_id(void* id_out);
amlt_status amlt_gpu_comm_attach(amlt_ctx* ctx, const void* id, int rank, int nranks);
amlt_status amlt_gpu_comm_detach(amlt_ctx* ctx);
/* Ranks of the attached communicator (1 when none). */
int amlt_gpu_comm_size(const amlt_ctx* ctx);

/* How the last amlt_gpu_run_host(_adaptive) call on ctx ran (diagnostics,
 * e.g. for a bench line): out[0] row bands, [1] K panels of B, [2] 1 when the
 * rows after band 0 wrote R straight into mapped host memory (zero-copy),
 * [3] rows of band 0, [4] k depth of the first panel, [5] 1 when B came by
 * broadcast, [6] 1 when the call tuned (whole task, no pipeline). */
#define AMLT_HOST_LAYOUT_FIELDS 7
amlt_status amlt_gpu_last_host_layout(const amlt_ctx* ctx, int64_t* out);

/* Row-band multi-GPU execution of one task from a single process (the
 * reference engine's process model). Device d of n owns rows
 * [i0 + M d/n, i0 + M (d+1)/n) of A and R; B and the per-column vectors are
 * copied to devices[0] once and replicated with one NCCL broadcast each over
 * NVLink / NVSwitch; there is no reduction (rows of R are independent). Each
 * device then runs amlt_gpu_adaptive_execute on its band (one host thread
 * per device) and its R rows are copied back. Operands are HOST buffers, as
 * for amlt_gpu_run_host; A must keep each row's k values contiguous
 * (A[i][k] row-major or A[k][i] col-major) and R must be row-major, so bands
 * are contiguous blocks (else UNSUPPORTED). NCCL (libnccl.so.2) is loaded at
 * run time. *elapsed_s covers copies, broadcast and compute. */
amlt_status amlt_gpu_run_sharded(const amlt_body_desc* desc, const amlt_operands* host_ops,
                                 const amlt_bounds* bounds, int n_devices, const int* devices,
                                 int flags, double* elapsed_s);
/* The same from a task text: any recognised statement, generated bodies
 * included (aux leaves bound by position as for amlt_gpu_plan_from_source).
 * Operands indexed by i follow the row split: row-major [i][j] leaves (and
 * thresholds) are copied band by band like R, [i] vectors are replicated
 * and viewed from the band's first row; [j] and scalar leaves are
 * replicated. */
amlt_status amlt_gpu_run_sharded_source(const char* task_source, int dtype,
                                        const amlt_operands* host_ops, const amlt_bounds* bounds,
                                        int n_devices, const int* devices, int flags,
                                        double* elapsed_s);
/* Message of the calling thread's last failing amlt_gpu_run_sharded(_source). */
const char* amlt_gpu_sharded_last_error(void);

/* The persistent form of amlt_gpu_run_sharded: a row-band group over n
 * devices of this process, made once (one context per device, one NCCL
 * communicator from ncclCommInitAll). Plans and tuning winners persist
 * across runs, so only the first run of a shape tunes. Each run: device d of
 * n owns rows [i0 + M d/n, i0 + M (d+1)/n) (edges on multiples of 64 rows);
 * every device runs the host pipeline of amlt_gpu_run_host_adaptive on its
 * band, device 0 reading B and the shared operands from host memory and
 * broadcasting them panel by panel (AMLT_HOST_BCAST_SHARED); R bands stream
 * back as they finish. The plan is `desc` when task_source is NULL, else the
 * task text (generated bodies included). reports: NULL or n entries, one per
 * device. *elapsed_s: wall time of the whole run. */
typedef struct amlt_sharded amlt_sharded;
/* ctx_flags AMLT_CTX_DRY_RUN: a group of device-less contexts (no NCCL);
 * runs plan and validate every band's operands and report each band's
 * rectangle (absolute rows) as its coverage, without computing. */
amlt_status amlt_sharded_create(int n_devices, const int* devices, int ctx_flags, amlt_sharded** out);
void amlt_sharded_destroy(amlt_sharded* group);
amlt_status amlt_sharded_run(amlt_sharded* group, const amlt_body_desc* desc, const char* task_source,
                             int dtype, const amlt_operands* host_ops, const amlt_bounds* bounds,
                             int flags, amlt_tune_report* reports, double* elapsed_s);
int amlt_sharded_size(const amlt_sharded* group);
/* Message of the group's last failing call (or of amlt_sharded_create when
 * group == NULL). Never NULL. */
const char* amlt_sharded_last_error(const amlt_sharded* group);

/* The reference's AMLT binary matrix files (README.md:146-157,
 * src/matrix.cpp:64-114; the CLI's --a-file / --b-file): 24-byte header
 * ("AMLT", u32 rows, u32 cols, u8 order, zero padding) then rows*cols f64
 * values in storage order. Reads convert to the requested dtype and can land
 * directly in device memory (chunked through a pinned buffer); writes
 * accept f64 / f32 / i32 host or device buffers in storage order. Errors:
 * ENGINE (bad magic, unknown order, truncated, unopenable), with the message
 * in amlt_matrix_file_last_error(). */
amlt_status amlt_matrix_file_info(const char* path, int64_t* rows, int64_t* cols, int* order);
amlt_status amlt_matrix_file_read(const char* path, void* dst, int dtype, int dst_on_device);
amlt_status amlt_matrix_file_write(const char* path, const void* src, int64_t rows, int64_t cols,
                                   int order, int dtype, int src_on_device);
const char* amlt_matrix_file_last_error(void);

/* The reference's seeded inputs (src/matrix.cpp:20-37, src/engine.cpp:147):
 * amlt_gen_matrix fills rows*cols values in storage order from mt19937_64
 * over seed_seq{seed, rows, cols, order, mode}; mode 0 = IntValued ([-8, 8]),
 * 1 = Real ([0, 1)). amlt_operand_seed(seed, name) = seed ^ fnv1a(name), the
 * per-array seed make_task_data uses. */
uint64_t amlt_operand_seed(uint64_t seed, const char* name);
amlt_status amlt_gen_matrix(uint64_t seed, int64_t rows, int64_t cols, int order, int mode,
                            void* dst, int dtype, int dst_on_device);

/* Pipe-throughput probe on the current device (roofline denominators):
 * pipe 0 DFMA, 1 FFMA, 2 integer ALU, 3 DSETP+select, 4 DMMA (f64 tensor).
 * *ops_per_s: lane operations per second (FMA pipes and DMMA: FMAs/s);
 * *sm_ghz: SM clock observed by the probe. */
amlt_status amlt_gpu_measure_peak(int pipe, double* ops_per_s, double* sm_ghz);

/* Scaled processing rate M*K*N / (1e9 * seconds) (engine.cpp:212-216). */
amlt_status amlt_spr(int64_t M, int64_t K, int64_t N, double seconds, double* out);

/* Device matrices for callers without an allocator of their own (the
 * reference hands over f64 MatrixBuffers). amlt_gpu_matrix_alloc returns a
 * rows x cols matrix in the given order and dtype whose leading dimension is
 * padded to 16 bytes (so the TMA-staged variants apply); upload / download
 * convert between the caller's f64 values (storage order, leading dimension
 * host_ld >= cols for row-major, >= rows for col-major) and the dtype.
 * Synchronous on the context stream. */
amlt_status amlt_gpu_matrix_alloc(amlt_ctx* ctx, int64_t rows, int64_t cols, int order, int dtype,
                                  amlt_matrix* out);
amlt_status amlt_gpu_matrix_free(amlt_ctx* ctx, amlt_matrix* m);
amlt_status amlt_gpu_matrix_upload(amlt_ctx* ctx, const amlt_matrix* dev, const double* host,
                                   int64_t host_ld);
amlt_status amlt_gpu_matrix_download(amlt_ctx* ctx, const amlt_matrix* dev, double* host,
                                     int64_t host_ld);

#ifdef __cplusplus
}
#endif

#endif /* AMLT_GPU_H */
