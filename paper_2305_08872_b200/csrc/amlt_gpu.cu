// amlt_gpu.cu — host side of the C-ABI in include/amlt_gpu.h.
//
// The executor (run_subtask), the runtime tuner (adaptive_execute) and the
// host-buffer entry of the B200 backend. Reference counterparts:
//   run_subtask        src/tiled_executor.cpp:9-77
//   adaptive_execute   src/autotuner.cpp:103-151 (find_kc :18-68, find_nc :70-101)
//   run_fixed/run_adaptive over host buffers   src/engine.cpp:165-175
// Errors are C++ exceptions internally (mirroring errors.hpp:10-60) and are
// mapped to amlt_status at the C boundary; the message is kept per context.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/amlt_gpu.h"
#include "jit.h"
#include "nccl_dl.h"
#include "naive.h"
#include "variants.h"

#include <cudaTypedefs.h>

using namespace amltk;

#include "task.h"

namespace {

// ---------------------------------------------------------------------------
// errors (errors.hpp:10-60)

struct EngineError : std::runtime_error {
    amlt_status code;
    EngineError(amlt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(amlt_status c, const std::string& m) { throw EngineError(c, m); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(AMLT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

thread_local std::string g_create_error = "";

const char* body_name(int b) {
    switch (b) {
        case AMLT_BODY_GEMM: return "gemm";
        case AMLT_BODY_DISCOUNT: return "discount";
        case AMLT_BODY_BOOST: return "boost";
        case AMLT_BODY_SQDIFF: return "sqdiff";
        case AMLT_BODY_EQCOUNT: return "eqcount";
        case AMLT_BODY_THRCOUNT: return "thrcount";
        case AMLT_BODY_GENERIC: return "generic";
    }
    return "?";
}
const char* dtype_name(int d) { return d == AMLT_F64 ? "f64" : d == AMLT_F32 ? "f32" : "i32"; }
int dtype_size(int d) { return d == AMLT_F64 ? 8 : 4; }

// ---------------------------------------------------------------------------
// registry of compiled variants (variants.h)

Registry& registry_storage() {
    static Registry reg;
    static std::once_flag once;
    std::call_once(once, [] { register_all(reg); });
    return reg;
}
const Registry& registry() { return registry_storage(); }

const BodyAux* find_aux(int body, int dtype) {
    std::lock_guard<std::mutex> lock(amltk::registry_mutex());
    for (const auto& a : registry().aux)
        if (a.body == body && a.dtype == dtype) return &a;
    return nullptr;
}

}  // namespace

namespace amltk {
Registry& registry_mut() { return registry_storage(); }
std::mutex& registry_mutex() {
    static std::mutex m;
    return m;
}
}  // namespace amltk

// ---------------------------------------------------------------------------
// context and plan

struct amlt_ctx {
    int device = 0;
    int flags = 0;
    int num_sms = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t hev0 = nullptr, hev1 = nullptr;  // host-entry call timing
    cudaStream_t copy_in = nullptr, copy_out = nullptr;  // run_host pipeline
    std::vector<cudaEvent_t> pipe_ev;                      // run_host pipeline
    void* work = nullptr;
    size_t work_bytes = 0;
    void* pack_ws = nullptr;  // dense copies of operands in other layouts
    size_t pack_bytes = 0;
    void* scratch = nullptr;  // scratch R for whole-task tuning trials
    size_t scratch_bytes = 0;
    void* tc_ws = nullptr;    // split / sliced operands of the tensor-core GEMMs
    size_t tc_ws_bytes = 0;
    // B's preparation in tc_ws, valid within one C-ABI call (call_gen)
    uint64_t call_gen = 0;
    // layout of the last host-pipeline call (amlt_gpu_last_host_layout)
    int64_t host_layout[AMLT_HOST_LAYOUT_FIELDS] = {};
    struct BPrep {
        const void* B = nullptr;
        int64_t ldb = 0, K = 0, N = 0;
        int prep = 0;
        uint64_t gen = ~uint64_t(0);
        const void* ws = nullptr;
        double seconds = 0.0;  // measured cost of the preparation (tuning trials)
    } bprep;
    // device staging for amlt_gpu_run_host
    // slots: A, B, R, thres, dis, then the aux leaves of generated bodies
    void* hbuf[5 + AMLT_MAX_AUX] = {};
    size_t hbuf_bytes[5 + AMLT_MAX_AUX] = {};
    mutable std::vector<int> occupancy;  // resident CTAs per SM, per registry variant (lazy for JIT)
    // tuning winners: (body, dtype, M, N, K) -> variant index
    struct Winner {
        int variant;
        int64_t kc;
        double row_seconds = 0.0;  // measured seconds per output row (0: unknown)
    };
    // keyed by (body, dtype, M, N, K, operands staging-aligned, variant family):
    // a winner only serves calls its variant can run
    using TuneKey = std::tuple<int, int, int64_t, int64_t, int64_t, int, int>;
    std::map<TuneKey, Winner> tune_cache;
    std::string err;
    // communicator of the multi-rank host entry (amlt_gpu_comm_attach, or a
    // rank of an amlt_sharded group): B and the replicated operands are
    // broadcast from rank 0 over NVLink / NVSwitch on comm_stream
    ncclComm_t comm = nullptr;
    bool comm_owned = false;
    int comm_rank = 0, comm_size = 1;
    cudaStream_t comm_stream = nullptr;
    bool dry() const { return (flags & AMLT_CTX_DRY_RUN) != 0; }
};

struct amlt_plan {
    amlt_body_desc desc{};
    std::vector<int> variants;  // registry indices usable for this body/dtype
    const BodyAux* aux = nullptr;
    const amlt_ctx* ctx = nullptr;
    // AMLT_BODY_GENERIC: the generated body's aux leaves, bound by position
    std::vector<std::string> aux_names;
    std::vector<int> aux_class;
};

namespace {

// ---------------------------------------------------------------------------
// operand validation (the GPU analogue of make_operands / find_aux,
// src/engine.cpp:153-163, src/kernel_exec.cpp:48-52)

// An operand region that must be packed into a dense row-major workspace.
struct Strided {
    const void* p = nullptr;
    int64_t rows = 0, cols = 0, s0 = 0, s1 = 0;
    bool need = false;
};

struct Resolved {
    KParams kp{};
    int64_t M = 0, N = 0, K = 0;
    bool aligned = true;  // 16-byte staging possible
    Strided pack_a, pack_b, pack_r;
    bool packed() const { return pack_a.need || pack_b.need || pack_r.need; }
};

// Element (r, c) of a statement operand with the given layout: returns the
// pointer of element (r0, c0) plus the strides along r and c, in elements.
void stmt_addr(const amlt_matrix& m, int layout, int64_t r0, int64_t c0, const char* what,
               char** ptr, int64_t* sr, int64_t* sc) {
    // statement (r, c) -> buffer (row, col)
    const bool tr = layout == AMLT_LAYOUT_TRANSPOSED;
    const int64_t brow = tr ? c0 : r0, bcol = tr ? r0 : c0;
    const int64_t es = dtype_size(m.dtype);
    const bool rowmaj = m.order == AMLT_ROW_MAJOR;
    const int64_t step_rows = rowmaj ? m.ld : 1;  // buffer row step
    const int64_t step_cols = rowmaj ? 1 : m.ld;
    *ptr = static_cast<char*>(m.data) + (brow * step_rows + bcol * step_cols) * es;
    *sr = tr ? step_cols : step_rows;
    *sc = tr ? step_rows : step_cols;
    (void)what;
}

void check_matrix(const amlt_matrix& m, int dtype, const char* what) {
    if (!m.data) fail(AMLT_ERR_MISSING_BINDING, std::string("missing binding for '") + what + "'");
    if (m.dtype != dtype)
        fail(AMLT_ERR_INVALID_ARGUMENT, std::string(what) + " has dtype " + dtype_name(m.dtype) +
                                            ", plan expects " + dtype_name(dtype));
    if (m.rows < 0 || m.cols < 0) fail(AMLT_ERR_INVALID_ARGUMENT, std::string(what) + ": negative shape");
    const int64_t minld = m.order == AMLT_ROW_MAJOR ? m.cols : m.rows;
    if (m.ld < std::max<int64_t>(minld, 1))
        fail(AMLT_ERR_INVALID_ARGUMENT, std::string(what) + ": leading dimension too small");
}

Resolved resolve(const amlt_plan* plan, const amlt_operands* ops, const amlt_bounds* b) {
    const amlt_body_desc& d = plan->desc;
    Resolved rv;
    KParams& kp = rv.kp;
    if (!ops || !b) fail(AMLT_ERR_INVALID_ARGUMENT, "null operands or bounds");
    rv.M = b->i1 - b->i0;
    rv.N = b->j1 - b->j0;
    rv.K = b->k1 - b->k0;
    if (rv.M < 0 || rv.N < 0 || rv.K < 0 || b->i0 < 0 || b->j0 < 0 || b->k0 < 0)
        fail(AMLT_ERR_INVALID_ARGUMENT, "bounds must be non-negative half-open ranges");
    check_matrix(ops->a, d.dtype, "A");
    check_matrix(ops->b, d.dtype, "B");
    check_matrix(ops->r, d.dtype, "R");
    const bool at = d.layout_a == AMLT_LAYOUT_TRANSPOSED, bt = d.layout_b == AMLT_LAYOUT_TRANSPOSED;
    // statement extents of each operand
    const int64_t a_i = at ? ops->a.cols : ops->a.rows, a_k = at ? ops->a.rows : ops->a.cols;
    const int64_t b_k = bt ? ops->b.cols : ops->b.rows, b_j = bt ? ops->b.rows : ops->b.cols;
    if (b->i1 > a_i || b->k1 > a_k || b->k1 > b_k || b->j1 > b_j || b->i1 > ops->r.rows ||
        b->j1 > ops->r.cols)
        fail(AMLT_ERR_INVALID_ARGUMENT, "bounds exceed an operand's extent");

    char *pa, *pb, *pr;
    int64_t sai, sak, sbk, sbj, sri, srj;
    stmt_addr(ops->a, d.layout_a, b->i0, b->k0, "A", &pa, &sai, &sak);
    stmt_addr(ops->b, d.layout_b, b->k0, b->j0, "B", &pb, &sbk, &sbj);
    stmt_addr(ops->r, AMLT_LAYOUT_NORMAL, b->i0, b->j0, "R", &pr, &sri, &srj);
    // The staged kernels read A along k and B / R along j contiguously. Any
    // other layout (transposed statements, col-major storage) is packed into
    // a dense row-major workspace first (packing.hpp:11-18), R also unpacked
    // after; the dense pitch is a multiple of 16 bytes (TMA).
    const int64_t vn16 = 16 / dtype_size(d.dtype);
    auto dense_ld = [&](int64_t cols) { return (std::max<int64_t>(cols, 1) + vn16 - 1) / vn16 * vn16; };
    kp.A = pa;
    kp.B = pb;
    kp.R = pr;
    kp.lda = sai;
    kp.ldb = sbk;
    kp.ldr = sri;
    if (sak != 1 && rv.K > 1) {
        rv.pack_a = {pa, rv.M, rv.K, sai, sak, true};
        kp.lda = dense_ld(rv.K);
    }
    if (sbj != 1 && rv.N > 1) {
        rv.pack_b = {pb, rv.K, rv.N, sbk, sbj, true};
        kp.ldb = dense_ld(rv.N);
    }
    if (srj != 1 && rv.N > 1) {
        rv.pack_r = {pr, rv.M, rv.N, sri, srj, true};
        kp.ldr = dense_ld(rv.N);
    }
    kp.M = rv.M;
    kp.N = rv.N;
    kp.K = rv.K;

    // aux leaves
    const bool needs_t = d.body == AMLT_BODY_DISCOUNT || d.body == AMLT_BODY_BOOST ||
                         d.body == AMLT_BODY_THRCOUNT;
    const bool needs_d = d.body == AMLT_BODY_DISCOUNT;
    kp.thres = nullptr;
    kp.tconst = d.thres_value;
    kp.t_si = 0;
    kp.t_sj = 0;
    const int64_t tes = dtype_size(d.dtype);
    // element step of a len x 1 (or 1 x len) vector buffer (kernel_exec.hpp:13-16)
    auto vec_step = [](const amlt_matrix& t) {
        return (t.cols == 1) ? (t.order == AMLT_ROW_MAJOR ? t.ld : 1)
                             : (t.order == AMLT_ROW_MAJOR ? 1 : t.ld);
    };
    if (needs_t && d.thres_class == AMLT_LEAF_CONSTANT && ops->thres.data) {
        // named scalar threshold (a 1 x 1 buffer): broadcast from device memory
        check_matrix(ops->thres, d.dtype, "thres");
        kp.thres = ops->thres.data;
    } else if (needs_t && d.thres_class == AMLT_LEAF_VEC_J) {
        check_matrix(ops->thres, d.dtype, "thres");
        const amlt_matrix& t = ops->thres;
        if (t.rows * t.cols < b->j1) fail(AMLT_ERR_INVALID_ARGUMENT, "thres shorter than j1");
        kp.t_sj = vec_step(t);
        kp.thres = static_cast<const char*>(t.data) + b->j0 * kp.t_sj * tes;
    } else if (needs_t && d.thres_class == AMLT_LEAF_VEC_I) {
        check_matrix(ops->thres, d.dtype, "thres");
        const amlt_matrix& t = ops->thres;
        if (t.rows * t.cols < b->i1) fail(AMLT_ERR_INVALID_ARGUMENT, "thres shorter than i1");
        kp.t_si = vec_step(t);
        kp.thres = static_cast<const char*>(t.data) + b->i0 * kp.t_si * tes;
    } else if (needs_t && d.thres_class == AMLT_LEAF_MAT_IJ) {
        check_matrix(ops->thres, d.dtype, "thres");
        const amlt_matrix& t = ops->thres;  // M x N, element (i, j)
        if (t.rows < b->i1 || t.cols < b->j1)
            fail(AMLT_ERR_INVALID_ARGUMENT, "thres[i][j] smaller than the bounds");
        kp.t_si = t.order == AMLT_ROW_MAJOR ? t.ld : 1;
        kp.t_sj = t.order == AMLT_ROW_MAJOR ? 1 : t.ld;
        kp.thres = static_cast<const char*>(t.data) + (b->i0 * kp.t_si + b->j0 * kp.t_sj) * tes;
    }
    kp.dis = nullptr;
    if (needs_d) {
        check_matrix(ops->dis, d.dtype, "dis");
        const amlt_matrix& t = ops->dis;
        if (t.rows * t.cols < b->j1) fail(AMLT_ERR_INVALID_ARGUMENT, "dis shorter than j1");
        const int64_t step = (t.cols == 1) ? (t.order == AMLT_ROW_MAJOR ? t.ld : 1)
                                           : (t.order == AMLT_ROW_MAJOR ? 1 : t.ld);
        kp.dis = static_cast<const char*>(t.data) + b->j0 * step * dtype_size(d.dtype);
        kp.d_sj = step;
    }

    // generated bodies: aux leaf q bound to ops->aux[q] by its index class
    for (int q = 0; q < AMLT_KP_MAX_AUX; ++q) {
        kp.gaux[q] = nullptr;
        kp.gaux_si[q] = 0;
        kp.gaux_sj[q] = 0;
    }
    if (d.body == AMLT_BODY_GENERIC) {
        const int nq = static_cast<int>(plan->aux_names.size());
        for (int q = 0; q < nq; ++q) {
            const std::string& nm = plan->aux_names[static_cast<size_t>(q)];
            if (q >= ops->n_aux || !ops->aux[q].data)
                fail(AMLT_ERR_MISSING_BINDING, "missing binding for '" + nm + "'");
            const amlt_matrix& t = ops->aux[q];
            check_matrix(t, d.dtype, nm.c_str());
            const int cls = plan->aux_class[static_cast<size_t>(q)];
            int64_t si = 0, sj = 0, off = 0;
            if (cls == AMLT_LEAF_CONSTANT) {
                if (t.rows * t.cols < 1) fail(AMLT_ERR_INVALID_ARGUMENT, nm + " is empty");
            } else if (cls == AMLT_LEAF_VEC_I) {
                if (t.rows * t.cols < b->i1) fail(AMLT_ERR_INVALID_ARGUMENT, nm + " shorter than i1");
                si = vec_step(t);
                off = b->i0 * si;
            } else if (cls == AMLT_LEAF_VEC_J) {
                if (t.rows * t.cols < b->j1) fail(AMLT_ERR_INVALID_ARGUMENT, nm + " shorter than j1");
                sj = vec_step(t);
                off = b->j0 * sj;
            } else {
                if (t.rows < b->i1 || t.cols < b->j1)
                    fail(AMLT_ERR_INVALID_ARGUMENT, nm + "[i][j] smaller than the bounds");
                si = t.order == AMLT_ROW_MAJOR ? t.ld : 1;
                sj = t.order == AMLT_ROW_MAJOR ? 1 : t.ld;
                off = b->i0 * si + b->j0 * sj;
            }
            kp.gaux[q] = static_cast<const char*>(t.data) + off * tes;
            kp.gaux_si[q] = si;
            kp.gaux_sj[q] = sj;
        }
    }

    const int es = dtype_size(d.dtype);
    const int vn = 16 / es;
    auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    // TMA staging: 16-byte aligned bases and row pitches
    // (packed operands land in a 256-byte aligned workspace)
    rv.aligned = (rv.pack_a.need || al16(kp.A)) && (rv.pack_b.need || al16(kp.B)) &&
                 kp.lda % vn == 0 && kp.ldb % vn == 0;
    kp.r_vec_ok = (rv.pack_r.need || al16(kp.R)) && (kp.ldr % vn == 0 || rv.M <= 1);
    return rv;
}

// ---------------------------------------------------------------------------
// variant choice

// Registry reads take the registry lock: run-time compiled bodies append
// entries from other threads (entries never move, so the reference stays valid).
const VariantDesc& vdesc(int idx) {
    std::lock_guard<std::mutex> lock(registry_mutex());
    return registry().variants.at(static_cast<size_t>(idx));
}

// Resident CTAs per SM of a registry variant on this context; computed on
// first use for variants added after the context was created (run-time
// compiled bodies).
int occ_of(const amlt_ctx* ctx, int idx) {
    const VariantDesc& v = vdesc(idx);
    if (!ctx) return v.minb;
    if (idx < static_cast<int>(ctx->occupancy.size()) && ctx->occupancy[static_cast<size_t>(idx)] > 0)
        return ctx->occupancy[static_cast<size_t>(idx)];
    int occ = v.minb;
    if (!ctx->dry() && v.func) {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, v.func, v.threads, v.smem) == cudaSuccess &&
            o > 0)
            occ = o;
        else
            (void)cudaGetLastError();
    }
    if (static_cast<int>(ctx->occupancy.size()) <= idx) ctx->occupancy.resize(static_cast<size_t>(idx) + 1, 0);
    ctx->occupancy[static_cast<size_t>(idx)] = occ;
    return occ;
}

int64_t ctas_for(const VariantDesc& v, int64_t M, int64_t N) {
    return ((M + v.bm - 1) / v.bm) * ((N + v.bn - 1) / v.bn);
}

// The planner's default: the largest tile that still fills every SM with at
// least two resident CTAs' worth of work; otherwise the variant with the most
// CTAs per wave slot (smallest tile).
int default_variant(const amlt_ctx* ctx, const amlt_plan* plan, int64_t M, int64_t N, bool aligned) {
    int best = -1;
    double best_key = -1;
    int fallback = -1;
    double fb_key = 1e300;
    for (int idx : plan->variants) {
        const VariantDesc& v = vdesc(idx);
        if (v.vec != aligned) continue;
        if (v.tc || v.run) continue;  // own staging + workspace: tuner candidates only
        const int occ = occ_of(ctx, idx);
        const int sms = ctx ? ctx->num_sms : 148;
        const double waves = double(ctas_for(v, M, N)) / double(sms * occ);
        const double area = double(v.bm) * v.bn;
        if (waves >= 2.0) {
            if (area > best_key) {
                best_key = area;
                best = idx;
            }
        }
        if (area < fb_key) {
            fb_key = area;
            fallback = idx;
        }
    }
    if (best >= 0) return best;
    if (fallback >= 0) return fallback;
    fail(AMLT_ERR_NO_FEASIBLE_KERNEL, std::string("no compiled tile variant for ") +
                                          body_name(plan->desc.body) + "/" +
                                          dtype_name(plan->desc.dtype));
}

int choose_variant(const amlt_ctx* ctx, const amlt_plan* plan, const amlt_tile_params* tile,
                   const Resolved& rv) {
    if (tile && tile->variant >= 0) {
        if (tile->variant >= (int)plan->variants.size())
            fail(AMLT_ERR_INVALID_ARGUMENT, "tile variant index out of range");
        int idx = plan->variants[static_cast<size_t>(tile->variant)];
        // (an empty rectangle runs nothing: no operand requirement applies)
        const bool empty = rv.M == 0 || rv.N == 0 || rv.K == 0;
        if (vdesc(idx).vec && !rv.aligned && !empty)
            fail(AMLT_ERR_INVALID_ARGUMENT,
                 "variant needs 16-byte aligned operands with vector-multiple strides");
        if (vdesc(idx).max_k && rv.K > vdesc(idx).max_k && !empty)
            fail(AMLT_ERR_INVALID_ARGUMENT, std::string("variant accepts K <= ") +
                                                std::to_string(vdesc(idx).max_k));
        return idx;
    }
    if (tile && tile->nc > 0) {
        int best = -1;
        for (int idx : plan->variants) {
            const VariantDesc& v = vdesc(idx);
            if (v.vec != rv.aligned || v.tc) continue;
            if (v.bn > tile->nc) continue;
            if (best < 0 || v.bn > vdesc(best).bn ||
                (v.bn == vdesc(best).bn && v.bm * v.tm > vdesc(best).bm * vdesc(best).tm))
                best = idx;
        }
        if (best >= 0) return best;
    }
    return default_variant(ctx, plan, rv.M, rv.N, rv.aligned);
}

amlt_ctx::TuneKey tune_key(const amlt_plan* plan, const Resolved& rv) {
    return amlt_ctx::TuneKey(plan->desc.body, plan->desc.dtype, rv.M, rv.N, rv.K, rv.aligned ? 1 : 0,
                             plan->variants.empty() ? -1 : plan->variants.front());
}

int plan_local_index(const amlt_plan* plan, int reg_idx) {
    for (size_t i = 0; i < plan->variants.size(); ++i)
        if (plan->variants[i] == reg_idx) return static_cast<int>(i);
    return -1;
}

// ---------------------------------------------------------------------------
// launch

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) fail(AMLT_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
    return fn;
}

void make_tensor_map(CUtensorMap* m, int dtype, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t row_bytes, int box_inner, int box_outer) {
    const CUtensorMapDataType dt = dtype == AMLT_F64   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                   : dtype == AMLT_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                       : CU_TENSOR_MAP_DATA_TYPE_INT32;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_outer)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = tensor_map_encoder()(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        fail(AMLT_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
}

void ensure_work(amlt_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->work_bytes) return;
    if (ctx->work) cudaFree(ctx->work);
    ctx->work = nullptr;
    ctx->work_bytes = 0;
    cuda_check(cudaMalloc(&ctx->work, bytes), "cudaMalloc(split-K workspace)");
    ctx->work_bytes = bytes;
}

struct Dispatch {
    int variant = -1;
    int splits = 1;
    int64_t kslice = 0;
};

Dispatch plan_dispatch(const amlt_ctx* ctx, const amlt_plan* plan, const amlt_tile_params* tile,
                       const Resolved& rv) {
    Dispatch dp;
    dp.variant = choose_variant(ctx, plan, tile, rv);
    dp.kslice = rv.K;
    if (tile && tile->kc > 0 && tile->kc < rv.K && (!vdesc(dp.variant).run || vdesc(dp.variant).splittable)) {
        // (variants with their own staging run the whole K range unless they
        // take K segments)
        // Segment starts stay multiples of 16 elements (one f64 k-tile, half
        // an f32 one) so every segment's operand rows keep the 16-byte
        // alignment the staged copies need and packed operands (4 k per
        // word) stay whole.
        const int64_t kc = (tile->kc + 15) / 16 * 16;
        dp.splits = static_cast<int>((rv.K + kc - 1) / kc);
        dp.kslice = kc;
        if (dp.splits > 65535) fail(AMLT_ERR_INVALID_ARGUMENT, "kc too small: more than 65535 K segments");
    }
    return dp;
}

void enqueue_compute(amlt_ctx* ctx, const amlt_plan* plan, Resolved& rv, const Dispatch& dp,
                     KParams kp);

// Workspace of the variants with their own staging, sized before any timed
// region (an allocation inside it would be charged to the trial).
void ensure_tc_ws(amlt_ctx* ctx, const VariantDesc& v, const KParams& kp) {
    if (!v.ws_bytes || ctx->dry()) return;
    const size_t need = v.ws_bytes(kp);
    if (need <= ctx->tc_ws_bytes) return;
    if (ctx->tc_ws) cudaFree(ctx->tc_ws);
    ctx->tc_ws = nullptr;
    ctx->tc_ws_bytes = 0;
    ctx->bprep.gen = ~uint64_t(0);
    cuda_check(cudaMalloc(&ctx->tc_ws, need), "cudaMalloc(tensor-core operand workspace)");
    ctx->tc_ws_bytes = need;
}

// Whether a variant's workspace (prepared B, split A, ...) can be allocated:
// what it needs beyond the current workspace must stay under 90% of free HBM
// with 1 GiB to spare.
bool ws_fits(const amlt_ctx* ctx, const VariantDesc& v, const KParams& kp) {
    if (!v.ws_bytes || ctx->dry()) return true;
    const size_t need = v.ws_bytes(kp);
    if (need <= ctx->tc_ws_bytes) return true;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    const double avail = 0.9 * double(free_b + ctx->tc_ws_bytes) - double(size_t(1) << 30);
    return double(need) <= avail;
}

bool bprep_ready(const amlt_ctx* ctx, const VariantDesc& v, const KParams& kp) {
    const auto& b = ctx->bprep;
    return b.gen == ctx->call_gen && b.prep == v.prep_id && b.B == kp.B && b.ldb == kp.ldb &&
           b.K == kp.K && b.N == kp.N && b.ws == ctx->tc_ws;
}
void bprep_mark(amlt_ctx* ctx, const VariantDesc& v, const KParams& kp, double seconds = 0.0) {
    ctx->bprep = amlt_ctx::BPrep{kp.B, kp.ldb, kp.K, kp.N, v.prep_id, ctx->call_gen, ctx->tc_ws, seconds};
}
// B's preparation ahead of a timed trial, so trials measure the per-band
// work; its own (event-timed) cost is kept in ctx->bprep.seconds, and the
// trial scores charge it back once per call (a cached winner pays it on
// every later call).
void prep_b_untimed(amlt_ctx* ctx, const VariantDesc& v, const KParams& kp) {
    if (!v.prep_b || ctx->dry()) return;
    ensure_tc_ws(ctx, v, kp);
    if (bprep_ready(ctx, v, kp)) return;
    // timed twice, the faster kept: a first run can pay one-off costs (cold
    // instruction cache, first use of the kernel) that no later call pays
    float best = 0;
    for (int rep = 0; rep < 2; ++rep) {
        cuda_check(cudaEventRecord(ctx->ev0, ctx->stream), "cudaEventRecord");
        cuda_check(v.prep_b(kp, ctx->tc_ws, ctx->stream), "tensor-core operand preparation");
        cuda_check(cudaEventRecord(ctx->ev1, ctx->stream), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(ctx->ev1), "cudaEventSynchronize");
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "cudaEventElapsedTime");
        best = rep == 0 ? ms : std::min(best, ms);
    }
    bprep_mark(ctx, v, kp, best * 1e-3);
}
// The preparation cost a trial of variant v leaves out (0 without one).
double prep_seconds(const amlt_ctx* ctx, const VariantDesc& v) {
    return v.prep_b && ctx->bprep.prep == v.prep_id && ctx->bprep.gen == ctx->call_gen ? ctx->bprep.seconds
                                                                                          : 0.0;
}

void enqueue(amlt_ctx* ctx, const amlt_plan* plan, Resolved& rv, const Dispatch& dp) {
    if (rv.M == 0 || rv.N == 0) return;
    if (rv.K == 0) return;  // empty k range: R untouched
    if (ctx->dry()) return;
    KParams kp = rv.kp;
    if (!rv.packed()) {
        enqueue_compute(ctx, plan, rv, dp, kp);
        return;
    }
    // Pack the operands the kernels cannot stage directly into one dense
    // row-major workspace (A, then B, then R), compute, unpack R.
    const size_t es = dtype_size(plan->desc.dtype);
    auto bytes_of = [&](const Strided& s, int64_t ld) {
        return s.need ? (size_t(s.rows) * size_t(ld) * es + 255) / 256 * 256 : size_t(0);
    };
    const size_t ba = bytes_of(rv.pack_a, kp.lda), bb = bytes_of(rv.pack_b, kp.ldb),
                 br = bytes_of(rv.pack_r, kp.ldr);
    if (ba + bb + br > ctx->pack_bytes) {
        if (ctx->pack_ws) cudaFree(ctx->pack_ws);
        ctx->pack_ws = nullptr;
        ctx->pack_bytes = 0;
        cuda_check(cudaMalloc(&ctx->pack_ws, ba + bb + br), "cudaMalloc(pack workspace)");
        ctx->pack_bytes = ba + bb + br;
    }
    char* w = static_cast<char*>(ctx->pack_ws);
    auto pack = [&](const Strided& s, void* dst, int64_t ld, int unpack) {
        PackParams pp{unpack ? dst : s.p, unpack ? const_cast<void*>(s.p) : dst, s.rows, s.cols,
                      s.s0, s.s1, ld, unpack};
        cuda_check(plan->aux->pack(pp, ctx->stream), "pack kernel launch");
    };
    if (rv.pack_a.need) {
        pack(rv.pack_a, w, kp.lda, 0);
        kp.A = w;
    }
    if (rv.pack_b.need) {
        pack(rv.pack_b, w + ba, kp.ldb, 0);
        kp.B = w + ba;
    }
    if (rv.pack_r.need) {
        pack(rv.pack_r, w + ba + bb, kp.ldr, 0);
        kp.R = w + ba + bb;
    }
    enqueue_compute(ctx, plan, rv, dp, kp);
    if (rv.pack_r.need) pack(rv.pack_r, w + ba + bb, kp.ldr, 1);
}

void enqueue_compute(amlt_ctx* ctx, const amlt_plan* plan, Resolved& rv, const Dispatch& dp,
                     KParams kp) {
    {
        const cudaError_t pend = cudaPeekAtLastError();
        if (pend != cudaSuccess)
            fail(AMLT_ERR_CUDA, std::string("stale CUDA error from an earlier call: ") +
                                    cudaGetErrorString(pend));
    }
    if (!plan->desc.accumulate) {
        // "=": only the last k term reaches R.
        const int64_t total = rv.M * rv.N;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 32));
        cuda_check(launch_helper_any(plan->aux->assign, plan->aux->assign_func, kp, dim3(blocks),
                                     ctx->stream),
                   "assign kernel launch");
        return;
    }
    const VariantDesc& v = vdesc(dp.variant);
    if (v.run) {  // own staging (tensor-core GEMMs, theta-form discount, packed eqcount)
        ensure_tc_ws(ctx, v, kp);
        const bool ready = bprep_ready(ctx, v, kp);
        kp.splits = 1;
        kp.kslice = rv.K;
        kp.work = nullptr;
        if (dp.splits > 1 && v.splittable) {
            kp.splits = dp.splits;
            kp.kslice = dp.kslice;
            ensure_work(ctx, size_t(dp.splits) * size_t(rv.M) * size_t(rv.N) * dtype_size(plan->desc.dtype));
            kp.work = ctx->work;
        }
        cuda_check(v.run(kp, ctx->tc_ws, ready, ctx->stream), "own-staging variant launch");
        if (!ready) bprep_mark(ctx, v, kp);
        if (kp.splits > 1) {
            const int64_t total = rv.M * rv.N;
            const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
            cuda_check(launch_helper_any(plan->aux->reduce, plan->aux->reduce_func, kp, dim3(blocks),
                                         ctx->stream),
                       "split-K reduce launch");
        }
        return;
    }
    kp.tiles_m = static_cast<int32_t>((rv.M + v.bm - 1) / v.bm);
    kp.tiles_n = static_cast<int32_t>((rv.N + v.bn - 1) / v.bn);
    kp.group_m = std::min(64, std::max(8, 512 / v.bm));
    const int64_t tiles = int64_t(kp.tiles_m) * kp.tiles_n;
    if (tiles > 0x7fffffffLL) fail(AMLT_ERR_INVALID_ARGUMENT, "problem too large for one launch");
    kp.splits = dp.splits;
    kp.kslice = dp.kslice;
    kp.work = nullptr;
    if (dp.splits > 1) {
        ensure_work(ctx, size_t(dp.splits) * size_t(rv.M) * size_t(rv.N) * dtype_size(plan->desc.dtype));
        kp.work = ctx->work;
    }
    CUtensorMap ma, mb;
    std::memset(&ma, 0, sizeof(ma));
    std::memset(&mb, 0, sizeof(mb));
    if (v.vec && !v.tc) {
        const int es = dtype_size(plan->desc.dtype);
        // A: inner dim k (K), outer dim i (M), box BK x BM; B: inner j (N),
        // outer k (K), box BN x BK. Zero fill outside the bounds rectangle.
        make_tensor_map(&ma, plan->desc.dtype, kp.A, uint64_t(rv.K), uint64_t(rv.M),
                        uint64_t(kp.lda) * es, v.bk, v.bm);
        make_tensor_map(&mb, plan->desc.dtype, kp.B, uint64_t(rv.N), uint64_t(rv.K),
                        uint64_t(kp.ldb) * es, v.bn, v.bk);
    }
    cuda_check(launch_tile_any(v, kp, ma, mb,
                               dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(dp.splits)),
                               ctx->stream),
               "tile kernel launch");
    if (dp.splits > 1) {
        const int64_t total = rv.M * rv.N;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
        cuda_check(launch_helper_any(plan->aux->reduce, plan->aux->reduce_func, kp, dim3(blocks),
                                     ctx->stream),
                   "split-K reduce launch");
    }
}

void log_dispatch(amlt_exec_log* log, const amlt_plan* plan, const Dispatch& dp,
                  const amlt_bounds& b) {
    if (!log) return;
    if (log->records && log->count < log->capacity) {
        amlt_exec_record& r = log->records[log->count++];
        r.variant = plan_local_index(plan, dp.variant);
        r.splits = dp.splits;
        r.i0 = b.i0; r.i1 = b.i1; r.j0 = b.j0; r.j1 = b.j1; r.k0 = b.k0; r.k1 = b.k1;
    }
    log->total++;
}

// One synchronous subtask, timed like run_subtask: exactly two clock reads
// around the work when a clock is given, CUDA events otherwise.
double timed_subtask(amlt_ctx* ctx, const amlt_plan* plan, Resolved& rv, const Dispatch& dp,
                     const amlt_bounds& b, amlt_clock_fn clock, void* user, amlt_exec_log* log) {
    double el = 0.0;
    if (!ctx->dry() && rv.M > 0 && rv.N > 0 && rv.K > 0 && !rv.packed())
        prep_b_untimed(ctx, vdesc(dp.variant), rv.kp);
    if (clock) {
        const double t0 = clock(user);
        enqueue(ctx, plan, rv, dp);
        if (!ctx->dry()) cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
        const double t1 = clock(user);
        el = t1 - t0;
    } else if (ctx->dry()) {
        el = 0.0;
    } else {
        cuda_check(cudaEventRecord(ctx->ev0, ctx->stream), "cudaEventRecord");
        enqueue(ctx, plan, rv, dp);
        cuda_check(cudaEventRecord(ctx->ev1, ctx->stream), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(ctx->ev1), "cudaEventSynchronize");
        float ms = 0.f;
        cuda_check(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "cudaEventElapsedTime");
        el = ms * 1e-3;
    }
    log_dispatch(log, plan, dp, b);
    return el;
}

Resolved resolve_sub(const amlt_plan* plan, const amlt_operands* ops, const amlt_bounds& b) {
    return resolve(plan, ops, &b);
}

// ---------------------------------------------------------------------------
// adaptive execution (autotuner.cpp:103-151, re-derived for a GPU)
//
// Candidates are the plan's tile variants (+ split-K forms when the output is
// too small to fill the GPU). Each candidate runs ONE row band of the real
// task (full N, full K), large enough to keep every SM busy for one wave,
// and is scored by elapsed / rows. The rest of the rows run with the winner.
// Every band writes its rows of R, so no work is repeated, and the coverage
// ledger proves every output is produced exactly once. A problem too small to
// give each candidate a full band runs whole with the planner default (or a
// winner cached from an earlier tuning of the same shape), like the
// reference's untuned small-task path (autotuner.cpp:112-122).

void add_cover(amlt_tune_report* rep, const amlt_bounds& b) {
    if (rep->n_cover < AMLT_MAX_COVER) {
        amlt_cover_rect& c = rep->coverage[rep->n_cover++];
        c.i0 = b.i0; c.i1 = b.i1; c.j0 = b.j0; c.j1 = b.j1; c.k0 = b.k0; c.k1 = b.k1;
    }
}

// Whole-task trials against a scratch R (see adaptive()). Records one trial
// per candidate (rows = M; score = elapsed / M) and caches the winner.
void scratch_tune(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                  const amlt_bounds& b, const Resolved& whole, const std::vector<int>& cands,
                  amlt_tune_report* rep) {
    const size_t bytes = size_t(whole.M) * size_t(whole.N) * dtype_size(plan->desc.dtype);
    if (bytes > ctx->scratch_bytes) {
        if (ctx->scratch) cudaFree(ctx->scratch);
        ctx->scratch = nullptr;
        ctx->scratch_bytes = 0;
        cuda_check(cudaMalloc(&ctx->scratch, bytes), "cudaMalloc(tuning scratch)");
        ctx->scratch_bytes = bytes;
    }
    struct Cand {
        int variant;
        int64_t kc;
    };
    std::vector<Cand> trials;
    for (int v : cands) {
        trials.push_back({v, 0});
        const VariantDesc& vd = vdesc(v);
        const int occ = occ_of(ctx, v);
        const int64_t ctas = ctas_for(vd, whole.M, whole.N);
        const int64_t slots = int64_t(ctx->num_sms) * occ;
        // split-K forms for small outputs (variants with their own staging run
        // whole K unless they take K segments)
        if ((!vd.run || vd.splittable) && ctas < 2 * slots && whole.K >= 512) {
            // K segments: 2, 3, 4, 6, 8, the count that fills two waves, and
            // the two counts (up to 16) whose CTAs come closest to whole waves
            // on this GPU (e.g. 88 tiles x 5 = 2.97 waves of 148); each
            // segment at least 128 deep. The measurement picks.
            std::vector<int64_t> counts = {2, 3, 4, 6, 8, (2 * slots + ctas - 1) / ctas};
            {
                std::vector<std::pair<double, int64_t>> eff;
                for (int64_t sp = 2; sp <= std::min<int64_t>(16, whole.K / 128); ++sp) {
                    const double waves = double(ctas * sp) / double(slots);
                    eff.push_back({-waves / std::ceil(waves), sp});
                }
                std::sort(eff.begin(), eff.end());
                for (size_t q = 0; q < eff.size() && q < 2; ++q) counts.push_back(eff[q].second);
            }
            std::vector<int64_t> kcs;
            for (int64_t splits : counts) {
                splits = std::min<int64_t>(splits, whole.K / 128);
                if (splits < 2) continue;
                const int64_t kc = ((whole.K + splits - 1) / splits + 15) / 16 * 16;
                if (std::find(kcs.begin(), kcs.end(), kc) == kcs.end()) kcs.push_back(kc);
            }
            for (int64_t kc : kcs) trials.push_back({v, kc});
        }
    }
    Resolved rs = resolve(plan, ops, &b);
    rs.kp.R = ctx->scratch;  // scratch R: dense row-major M x N
    rs.kp.ldr = whole.N;
    rs.kp.r_vec_ok = (whole.N * dtype_size(plan->desc.dtype)) % 16 == 0;
    rs.pack_r = Strided{};
    double best_t = 0;
    Cand best{-1, 0};
    for (const Cand& c : trials) {
        amlt_tile_params tp{c.kc, 0, 0, plan_local_index(plan, c.variant)};
        Dispatch dp = plan_dispatch(ctx, plan, &tp, rs);
        if (!rs.packed()) prep_b_untimed(ctx, vdesc(dp.variant), rs.kp);
        else ensure_tc_ws(ctx, vdesc(dp.variant), rs.kp);
        // two runs, the faster scored: the first can pay one-off costs (cold
        // instruction cache, first launch of the kernel) the cached winner
        // never pays again; all are charged to the call. Sub-millisecond
        // tasks take five: their candidates sit within a few percent of each
        // other (config 0), and two runs let launch jitter pick the winner.
        float ms = 0, ms_sum = 0;
        int reps = 2;
        for (int rep = 0; rep < reps; ++rep) {
            cuda_check(cudaEventRecord(ctx->ev0, ctx->stream), "cudaEventRecord");
            enqueue(ctx, plan, rs, dp);
            cuda_check(cudaEventRecord(ctx->ev1, ctx->stream), "cudaEventRecord");
            cuda_check(cudaEventSynchronize(ctx->ev1), "cudaEventSynchronize");
            float one = 0;
            cuda_check(cudaEventElapsedTime(&one, ctx->ev0, ctx->ev1), "cudaEventElapsedTime");
            ms = rep == 0 ? one : std::min(ms, one);
            ms_sum += one;
            if (rep == 0 && one < 1.0f) reps = 5;
        }
        // the whole task: its B preparation is part of every call
        const double el = ms * 1e-3 + (rs.packed() ? 0.0 : prep_seconds(ctx, vdesc(dp.variant)));
        if (rep->n_trials < AMLT_MAX_TRIALS) {
            amlt_trial& t = rep->trials[rep->n_trials++];
            t.value = plan_local_index(plan, c.variant);
            t.rows = whole.M;
            t.elapsed = el;
            t.score = el / double(whole.M);
        }
        // the trials' work is repeated for the real R: charged to the call
        const double spent = ms_sum * 1e-3 + (rs.packed() ? 0.0 : prep_seconds(ctx, vdesc(dp.variant)));
        rep->tuning_seconds += spent;
        rep->total_seconds += spent;
        if (best.variant < 0 || el < best_t) {
            best_t = el;
            best = c;
        }
    }
    rep->scratch_tuned = 1;
    ctx->tune_cache[tune_key(plan, whole)] =
        amlt_ctx::Winner{best.variant, best.kc, best_t / double(std::max<int64_t>(whole.M, 1))};
}

void adaptive(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops, const amlt_bounds& b,
              amlt_clock_fn clock, void* user, amlt_exec_log* log, amlt_tune_report* rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->best_variant = -1;
    Resolved whole = resolve(plan, ops, &b);
    const auto key = tune_key(plan, whole);

    // candidate list
    std::vector<int> cands;
    for (int idx : plan->variants) {
        const VariantDesc& v = vdesc(idx);
        if (v.emulated && !(ctx->flags & AMLT_CTX_F64_EMULATION)) continue;  // opt-in only
        if (v.max_k && whole.K > v.max_k) continue;
        if (!ws_fits(ctx, v, whole.kp)) continue;  // prepared operands would not fit in HBM
        if (v.vec == whole.aligned && (!v.tc || whole.aligned)) cands.push_back(idx);
    }
    // Band height per candidate: `waves` full waves of CTAs across all SMs
    // (8 when the rows allow it, else 4, so partial-wave tails weigh little
    // in the score; otherwise 1). At config 4's shape 4-wave bands ranked the
    // 96 x 128 theta tile 0.6% ahead of the 48 x 128 one, which is 1.3%
    // faster over whole launches (tools/theta_variants.py).
    // The bands must fit in a quarter of the rows (8-, 4-, then 1-wave bands).
    // Tasks small enough are better measured whole on a scratch R (below);
    // for larger ones with many candidates, 1-wave bands may take up to 40%
    // of the rows (their rows are real output, computed by the candidate
    // under trial).
    const bool scratch_ok = double(whole.M) * double(whole.N) * double(whole.K) <= 1.5e11 &&
                            whole.M * whole.N * dtype_size(plan->desc.dtype) <= (int64_t(1) << 30);
    std::vector<int64_t> band(cands.size());
    int64_t need = 0;
    int64_t cap = whole.M / 4;
    int used_waves = 8;
    for (int attempt = 0; attempt < (scratch_ok ? 3 : 4); ++attempt) {
        const int waves = attempt == 0 ? 8 : attempt == 1 ? 4 : 1;
        used_waves = waves;
        cap = attempt < 3 ? whole.M / 4 : whole.M * 2 / 5;
        need = 0;
        for (size_t c = 0; c < cands.size(); ++c) {
            const VariantDesc& v = vdesc(cands[c]);
            const int occ = occ_of(ctx, cands[c]);
            // (an empty N leaves no tiles: one-row bands; the task is then
            // not tunable and runs through the untuned path below)
            const int64_t tiles_n = std::max<int64_t>(1, (whole.N + v.bn - 1) / v.bn);
            const int64_t want_ctas = int64_t(waves) * ctx->num_sms * occ;
            const int64_t tiles_m = std::max<int64_t>(1, (want_ctas + tiles_n - 1) / tiles_n);
            band[c] = tiles_m * v.bm;
            need += band[c];
        }
        if (need <= cap) break;
    }
    // Tasks cheap enough to repeat are measured whole on the scratch R even
    // when row bands would fit: a band of a few waves sees a different L2
    // (its B panels stay resident, the whole task's do not), and at config
    // 1's shape that misranked the tiles by up to 12% (tools/tuner_stability.py,
    // profiles/r01/tuner_stability.txt). A caller-supplied clock keeps the
    // band trials: its readings are the AMULET contract's scores.
    const bool prefer_scratch = scratch_ok && !clock && !ctx->dry();
    const bool tunable = !prefer_scratch && plan->desc.accumulate && !cands.empty() && whole.K > 0 &&
                         whole.N > 0 && whole.M > 0 && need <= cap && ctx->tune_cache.find(key) == ctx->tune_cache.end();

    auto run_rect = [&](const amlt_bounds& rb, int variant, int64_t kc) {
        amlt_tile_params tp{kc, 0, 0, plan_local_index(plan, variant)};
        Resolved rv = resolve_sub(plan, ops, rb);
        Dispatch dp = plan_dispatch(ctx, plan, &tp, rv);
        double el = timed_subtask(ctx, plan, rv, dp, rb, clock, user, log);
        rep->total_seconds += el;
        add_cover(rep, rb);
        return el;
    };

    // Too small for row-band trials (each candidate would need more than a
    // quarter of the rows to fill the GPU): measure every candidate — tile
    // variants, plus split-K forms when the output cannot fill the SMs — on
    // the whole task against a scratch R, once per shape; the winner is
    // cached and the real task runs once with it. Skipped in dry-run
    // contexts and for tasks too large to repeat cheaply.
    if (!tunable && plan->desc.accumulate && !ctx->dry() && !cands.empty() && whole.M > 0 &&
        whole.N > 0 && whole.K > 0 && ctx->tune_cache.find(key) == ctx->tune_cache.end() &&
        scratch_ok) {
        scratch_tune(ctx, plan, ops, b, whole, cands, rep);
    }
    if (!tunable) {
        rep->tuned = 0;
        auto it = ctx->tune_cache.find(key);
        int v;
        int64_t kc = 0;
        if (it != ctx->tune_cache.end()) {
            // a winner measured on an earlier call with the same shape (or
            // by this call's scratch trials just above: not from the cache)
            v = it->second.variant;
            kc = it->second.kc;
            rep->from_cache = rep->scratch_tuned ? 0 : 1;
        } else if (!plan->desc.accumulate) {
            // "=" runs the per-element assign kernel; any staging-compatible variant
            v = default_variant(ctx, plan, whole.M, whole.N, whole.aligned);
        } else {
            v = default_variant(ctx, plan, whole.M, whole.N, whole.aligned);
            // Output too small to fill the GPU: split K so every SM has work
            // (per-segment partials are reduced in order: deterministic).
            const VariantDesc& vd = vdesc(v);
            const int occ = occ_of(ctx, v);
            const int64_t ctas = ctas_for(vd, whole.M, whole.N);
            const int64_t slots = int64_t(ctx->num_sms) * occ;
            if (ctas > 0 && ctas < slots && whole.K >= 512) {
                int64_t splits = std::min<int64_t>((slots + ctas - 1) / ctas, whole.K / 256);
                if (splits > 1) kc = ((whole.K + splits - 1) / splits + 15) / 16 * 16;
            }
        }
        rep->best_variant = v >= 0 ? plan_local_index(plan, v) : -1;
        rep->best_kc = kc > 0 ? kc : whole.K;
        if (whole.M > 0 && whole.N > 0) run_rect(b, v < 0 ? plan->variants[0] : v, kc);
        else add_cover(rep, b);
        rep->tuning_fraction = 0.0;
        return;
    }

    rep->tuned = 1;
    int64_t cur = b.i0;
    int best = -1;
    double best_score = 0.0;
    std::vector<std::pair<double, int>> scored;  // (score, candidate) of the first pass
    // one trial band: its rows are real output; the score is seconds per row
    auto trial_band = [&](int cand, int64_t rows) {
        amlt_bounds rb{cur, cur + rows, b.j0, b.j1, b.k0, b.k1};
        double el = run_rect(rb, cand, 0);
        amlt_trial& t = rep->trials[rep->n_trials++];
        t.value = plan_local_index(plan, cand);
        t.rows = rows;
        t.elapsed = el;
        // A band cannot hold a whole number of waves for every tile shape
        // (e.g. 3 x 256 CTAs of 96 x 128 on 148 SMs is 5.19 CTAs per SM,
        // run as 6): score the band as if its busiest SM's last CTA round
        // were full, which is what the many-wave remainder sees.
        const VariantDesc& v = vdesc(cand);
        const double per_sm = double(ctas_for(v, rows, whole.N)) / double(ctx->num_sms);
        const double full = per_sm > 0.0 ? per_sm / std::ceil(per_sm) : 1.0;
        // plus the variant's B preparation spread over the whole task
        t.score = el * full / double(rows) + prep_seconds(ctx, v) / double(whole.M);
        cur += rows;
        return t.score;
    };
    for (size_t c = 0; c < cands.size() && rep->n_trials < AMLT_MAX_TRIALS; ++c) {
        const double sc = trial_band(cands[c], band[c]);
        scored.push_back({sc, cands[c]});
        if (best < 0 || sc < best_score) {
            best = cands[c];
            best_score = sc;
        }
    }
    // Bands shorter than 8 waves (the rows did not allow more) misrank
    // near-equal tiles: at 4096 rows of config 4's columns the 1-wave bands
    // put the 96 x 128 theta tile first, 1.6% slower than the 48 x 128 one
    // over the whole band (bench.py --proxy-band 8). Then the best three (or
    // two, when three do not fit in the rows left) run one more band each at
    // 8 waves, real rows again, and the best of those wins. Device-timed calls
    // only: a caller's clock scripts the first pass.
    if (!clock && used_waves < 8 && scored.size() >= 2) {
        std::sort(scored.begin(), scored.end());
        auto rows8 = [&](int cand) {
            const VariantDesc& v = vdesc(cand);
            const int64_t tiles_n = std::max<int64_t>(1, (whole.N + v.bn - 1) / v.bn);
            const int64_t want_ctas = int64_t(8) * ctx->num_sms * occ_of(ctx, cand);
            return std::max<int64_t>(1, (want_ctas + tiles_n - 1) / tiles_n) * v.bm;
        };
        for (size_t top = std::min<size_t>(3, scored.size()); top >= 2; --top) {
            int64_t need8 = 0;
            for (size_t q = 0; q < top; ++q) need8 += rows8(scored[q].second);
            if (cur + need8 > b.i1 || rep->n_trials + int(top) > AMLT_MAX_TRIALS) continue;
            best = -1;
            for (size_t q = 0; q < top; ++q) {
                const int cand = scored[q].second;
                const double sc = trial_band(cand, rows8(cand));
                if (best < 0 || sc < best_score) {
                    best = cand;
                    best_score = sc;
                }
            }
            rep->refined = int32_t(top);
            break;
        }
    }
    rep->best_variant = plan_local_index(plan, best);
    rep->best_kc = whole.K;
    rep->tuning_fraction = double(cur - b.i0) / double(whole.M);
    ctx->tune_cache[key] = amlt_ctx::Winner{best, 0, best_score};
    if (cur < b.i1) run_rect(amlt_bounds{cur, b.i1, b.j0, b.j1, b.k0, b.k1}, best, 0);
}

// ---------------------------------------------------------------------------
// AMULET's tuner contract (src/autotuner.cpp:8-151), restated over the GPU
// executor. Decisions depend only on the clock readings, so a scripted clock
// reproduces the reference's kc / nc choices exactly.

struct AmuletTuner {
    amlt_ctx* ctx;
    const amlt_plan* plan;
    const amlt_operands* ops;
    amlt_clock_fn clock;
    void* user;
    amlt_exec_log* log;
    amlt_amulet_report* rep;

    // run_subtask with TileParams{kc, nc}
    double sub(const amlt_bounds& b, int64_t kc, int64_t nc) {
        amlt_tile_params tp{kc, nc, 0, -1};
        Resolved rv = resolve(plan, ops, &b);
        Dispatch dp = plan_dispatch(ctx, plan, &tp, rv);
        double el = timed_subtask(ctx, plan, rv, dp, b, clock, user, log);
        rep->total_seconds += el;
        return el;
    }
    void cover(int64_t k0, int64_t k1, int64_t j0, int64_t j1) {
        if (rep->n_cover < AMLT_MAX_REF_COVER) rep->coverage[rep->n_cover++] = {k0, k1, j0, j1};
    }
    static void trial(amlt_ref_trial* arr, int32_t* n, int64_t v, double el) {
        if (*n < AMLT_MAX_REF_TRIALS) arr[(*n)++] = {v, el, el / double(v)};
    }
    // kc_candidates (autotuner.cpp:8-16)
    static std::vector<int64_t> kc_candidates(int64_t K) {
        std::vector<int64_t> out;
        if (K < 16) {
            out.push_back(K);
            return out;
        }
        for (int64_t c = K; c >= 16; c = (c + 1) / 2) out.push_back(c);
        return out;
    }
    int64_t best_kc_so_far(const std::vector<int64_t>& cands) const {
        int64_t best = cands[0];
        double best_score = rep->n_kc_trials ? rep->kc_trials[0].score : 0.0;
        for (int t = 0; t < rep->n_kc_trials; ++t)
            if (rep->kc_trials[t].score < best_score) {
                best_score = rep->kc_trials[t].score;
                best = rep->kc_trials[t].value;
            }
        return best;
    }
    // find_kc (autotuner.cpp:18-68)
    int64_t find_kc(const amlt_bounds& b, int64_t iw) {
        const auto cands = kc_candidates(b.k1 - b.k0);
        {
            amlt_bounds s1{b.i0, b.i1, b.j0, b.j0 + 2 * iw, b.k0, b.k1};
            double el = sub(s1, cands[0], iw);
            trial(rep->kc_trials, &rep->n_kc_trials, cands[0], el);
            cover(b.k0, b.k1, s1.j0, s1.j1);
        }
        const int64_t sj0 = b.j0 + 2 * iw, sj1 = b.j0 + 4 * iw;
        int64_t kcur = b.k0;
        for (size_t ci = 1; ci < cands.size(); ++ci) {
            const int64_t len = cands[ci];
            if (kcur + len > b.k1) continue;
            double el = sub(amlt_bounds{b.i0, b.i1, sj0, sj1, kcur, kcur + len}, len, iw);
            trial(rep->kc_trials, &rep->n_kc_trials, len, el);
            cover(kcur, kcur + len, sj0, sj1);
            kcur += len;
        }
        if (kcur < b.k1) {
            sub(amlt_bounds{b.i0, b.i1, sj0, sj1, kcur, b.k1}, best_kc_so_far(cands), iw);
            cover(kcur, b.k1, sj0, sj1);
        }
        return best_kc_so_far(cands);
    }
    // find_nc (autotuner.cpp:70-101)
    int64_t find_nc(const amlt_bounds& b, int64_t best_kc, int64_t iw) {
        int64_t jcur = b.j0 + 4 * iw;
        const int64_t kb1 = std::min(b.k0 + best_kc, b.k1);
        int64_t best = 0, prev = 0;
        double best_score = 0.0, prev_score = 0.0;
        for (int64_t w = iw;; w *= 2) {
            if (jcur + w > b.j1) break;
            double el = sub(amlt_bounds{b.i0, b.i1, jcur, jcur + w, b.k0, kb1}, best_kc, w);
            const double score = el / double(w);
            trial(rep->nc_trials, &rep->n_nc_trials, w, el);
            cover(b.k0, kb1, jcur, jcur + w);
            jcur += w;
            if (prev != 0 && score > prev_score) return prev;
            prev = w;
            prev_score = score;
            if (best == 0 || score < best_score) {
                best = w;
                best_score = score;
            }
        }
        return best != 0 ? best : b.j1 - b.j0;
    }
    // adaptive_execute (autotuner.cpp:103-151)
    void run(const amlt_bounds& b, int64_t ih, int64_t iw) {
        const int64_t N = b.j1 - b.j0, K = b.k1 - b.k0;
        if (N < 4 * iw || b.i1 - b.i0 < ih) {
            rep->tuned = 0;
            rep->best_kc = std::min<int64_t>(K, 256);
            rep->best_nc = N;
            sub(b, rep->best_kc, rep->best_nc);
            cover(b.k0, b.k1, b.j0, b.j1);
            rep->tuning_fraction = 0.0;
            return;
        }
        rep->tuned = 1;
        rep->best_kc = find_kc(b, iw);
        rep->best_nc = find_nc(b, rep->best_kc, iw);
        int64_t tested_w = 0;
        for (int t = 0; t < rep->n_nc_trials; ++t) tested_w += rep->nc_trials[t].value;
        rep->tuning_fraction = double(4 * iw + tested_w) / double(N);
        const int64_t nc_j0 = b.j0 + 4 * iw, nc_j1 = nc_j0 + tested_w;
        const int64_t kb1 = std::min(b.k0 + rep->best_kc, b.k1);
        if (tested_w > 0 && kb1 < b.k1) {
            sub(amlt_bounds{b.i0, b.i1, nc_j0, nc_j1, kb1, b.k1}, rep->best_kc, rep->best_nc);
            cover(kb1, b.k1, nc_j0, nc_j1);
        }
        if (nc_j1 < b.j1) {
            sub(amlt_bounds{b.i0, b.i1, nc_j1, b.j1, b.k0, b.k1}, rep->best_kc, rep->best_nc);
            cover(b.k0, b.k1, nc_j1, b.j1);
        }
    }
};


// ---------------------------------------------------------------------------
// communicator of the multi-rank host entry

void comm_release(amlt_ctx* ctx) {
    if (ctx->comm && ctx->comm_owned) nccl().destroy(ctx->comm);
    ctx->comm = nullptr;
    ctx->comm_owned = false;
    ctx->comm_rank = 0;
    ctx->comm_size = 1;
}

void comm_use(amlt_ctx* ctx, ncclComm_t c, int rank, int n, bool owned) {
    comm_release(ctx);
    ctx->comm = c;
    ctx->comm_owned = owned;
    ctx->comm_rank = rank;
    ctx->comm_size = n;
    if (!ctx->comm_stream)
        cuda_check(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking), "cudaStreamCreate");
}

void nccl_check(int r, const char* what) {
    if (r != kNcclSuccess) fail(AMLT_ERR_CUDA, std::string(what) + ": " + nccl_error_string(r));
}

// ---------------------------------------------------------------------------
// The host-buffer entry (run_fixed / run_adaptive over host MatrixBuffers,
// src/engine.cpp:165-175): a copy / compute pipeline over row bands of A and
// R and K panels of B.
//
//   copy_in   : replicated operands, A band 0 (+ R band 0), B panel 0, the
//               other A bands, the other B panels (H2D)
//   comm      : with a communicator and AMLT_HOST_BCAST_SHARED, rank 0's B
//               panels and replicated operands are broadcast (NCCL) as they land
//   compute   : for each K panel p, for each row band b: R[b] += body over
//               k in panel p (the kernels accumulate into R)
//   copy_out  : R band b (D2H) as soon as its last panel is done
//
// Compute starts as soon as the first band of A and the first panel of B are
// resident; later transfers overlap it. Panels need B's k rows contiguous
// (B[k][j] row-major or B[j][k] col-major) and are skipped for split-K
// winners and "=" statements. With `rep` and no tuned winner for the shape,
// the whole task is copied first and runs through the tuner (adaptive).

int host_ncopies(const amlt_operands* ho) { return 5 + std::max(0, std::min<int>(ho->n_aux, AMLT_MAX_AUX)); }

// Is operand slot s (0 A, 1 B, 2 R, 3 thres, 4 dis, 5+ aux) replicated on
// every rank (as opposed to indexed by the rank's rows)?
bool slot_replicated(const amlt_plan* plan, int s) {
    auto rep_class = [](int c) { return c == AMLT_LEAF_CONSTANT || c == AMLT_LEAF_VEC_J; };
    if (s == 1) return true;
    if (s == 3) return rep_class(plan->desc.thres_class);
    if (s == 4) return true;
    if (s >= 5) {
        const size_t q = static_cast<size_t>(s - 5);
        return q < plan->aux_class.size() && rep_class(plan->aux_class[q]);
    }
    return false;
}

std::vector<int64_t> band_edges(int64_t lo, int64_t n, int nb, int64_t align, bool short_last) {
    std::vector<int64_t> e(static_cast<size_t>(nb) + 1);
    for (int b = 0; b <= nb; ++b) {
        double f = nb == 1 ? double(b) : (short_last ? std::min(1.0, b / (nb - 0.875)) : double(b) / nb);
        int64_t r = static_cast<int64_t>(f * double(n));
        if (b < nb) r = r / align * align;
        e[static_cast<size_t>(b)] = lo + std::min<int64_t>(n, b == nb ? n : r);
    }
    return e;
}

void host_pipeline(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* host_ops,
                   const amlt_tile_params* tile, const amlt_bounds* bounds, int flags, amlt_clock_fn clock,
                   void* clock_user, amlt_tune_report* rep, double* elapsed_s) {
    if (ctx->dry()) fail(AMLT_ERR_NO_DEVICE, "amlt_gpu_run_host needs a device context");
    cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
    const amlt_body_desc& d = plan->desc;
    const int es = dtype_size(d.dtype);
    const bool r_zero = (flags & AMLT_HOST_R_ZERO) != 0;
    const bool bcast = (flags & AMLT_HOST_BCAST_SHARED) != 0 && ctx->comm;
    const bool root = !bcast || ctx->comm_rank == 0;
    const int nslot = host_ncopies(host_ops);

    // Host view for validation. Off the root, replicated operands arrive by
    // broadcast: their shapes must be given, their data may be NULL.
    amlt_operands hview = *host_ops;
    amlt_matrix* hslot[5 + AMLT_MAX_AUX] = {&hview.a, &hview.b, &hview.r, &hview.thres, &hview.dis};
    for (int q = 0; q + 5 < nslot; ++q) hslot[5 + q] = &hview.aux[q];
    std::vector<bool> shared(static_cast<size_t>(nslot), false);
    for (int s = 0; s < nslot; ++s) {
        shared[static_cast<size_t>(s)] = slot_replicated(plan, s);
        if (bcast && !root && shared[static_cast<size_t>(s)] && !hslot[s]->data && hslot[s]->rows > 0)
            hslot[s]->data = reinterpret_cast<void*>(uintptr_t(256));  // shape only; never read here
    }
    Resolved hv = resolve(plan, &hview, bounds);

    // each operand's host extent: (outer - 1) whole pitches plus one inner run
    // (a view into a larger host buffer never reads past its own end)
    size_t bytes[5 + AMLT_MAX_AUX] = {};
    for (int s = 0; s < nslot; ++s) {
        const amlt_matrix& m = *hslot[s];
        if (!m.data) continue;
        const int64_t outer = m.order == AMLT_ROW_MAJOR ? m.rows : m.cols;
        const int64_t inner = m.order == AMLT_ROW_MAJOR ? m.cols : m.rows;
        bytes[s] = outer > 0 && inner > 0 ? (size_t(outer - 1) * size_t(m.ld) + size_t(inner)) * es : 0;
    }

    // the variant: the caller's tile, else the winner cached for this shape,
    // else (rep given) tune now, else the planner default
    amlt_tile_params tp{0, 0, 0, -1};
    const auto key = tune_key(plan, hv);
    bool cached = false;
    double row_seconds = 0.0;
    {
        auto it = ctx->tune_cache.find(key);
        if (tile) {
            tp = *tile;
        } else if (it != ctx->tune_cache.end()) {
            tp.variant = plan_local_index(plan, it->second.variant);
            tp.kc = it->second.kc;
            row_seconds = it->second.row_seconds;
            cached = true;
        }
    }
    const bool tune_now = rep && !tile && !cached;
    const int64_t M = hv.M, N = hv.N, K = hv.K;
    const int vi = !tune_now ? (tp.variant >= 0 ? plan->variants[static_cast<size_t>(tp.variant)]
                                                : default_variant(ctx, plan, M, N, hv.aligned))
                             : -1;

    // row bands of A / R (A rows k-contiguous, R row-major)
    const bool a_rows = (d.layout_a == AMLT_LAYOUT_NORMAL && host_ops->a.order == AMLT_ROW_MAJOR);
    const bool r_rows = host_ops->r.order == AMLT_ROW_MAJOR;
    // K panels of B (B's k rows contiguous)
    const bool b_kouter = (d.layout_b == AMLT_LAYOUT_NORMAL && host_ops->b.order == AMLT_ROW_MAJOR) ||
                          (d.layout_b == AMLT_LAYOUT_TRANSPOSED && host_ops->b.order == AMLT_COL_MAJOR);
    const bool split_winner = tp.kc > 0 && tp.kc < K;
    const bool banded = !tune_now && a_rows && r_rows && M >= 1024;

    // Result straight to the host: when R is pinned host memory the device
    // can address (cudaHostAlloc / cudaHostRegister, mapped), the rows after
    // band 0 run as ONE launch whose epilogue stores R into host memory over
    // PCIe (and, without R_ZERO, reads it from there): each R element crosses
    // the bus once, as the D2H copy would have, with no copy-out stage, no
    // staging buffer and no band boundaries after band 0. Needs a variant
    // whose epilogue (and split-K reduce) does plain global stores and
    // honours KParams::r_zero, whole-K launches, and no packing of R.
    // AMLT_HOST_NO_ZEROCOPY=1 keeps the staged pipeline (diagnostics).
    void* r_mapped = nullptr;
    if (banded && d.accumulate && vi >= 0 && vdesc(vi).r_overwrite && !std::getenv("AMLT_HOST_NO_ZEROCOPY")) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, host_ops->r.data) == cudaSuccess) {
            if (at.type == cudaMemoryTypeHost && at.devicePointer) r_mapped = at.devicePointer;
        } else {
            (void)cudaGetLastError();  // unregistered pageable memory: staged pipeline
        }
    }

    // (the panel count depends only on what every rank of a broadcast shares,
    // so all ranks issue the same sequence of collectives)
    // Panels of at least 4 MiB of B (AMLT_HOST_PANEL_BYTES overrides; tests
    // use it to cut small tasks) and 256 k, at most 8.
    int np = 1;
    if (b_kouter && d.accumulate) {
        double panel_bytes = double(4 << 20);
        if (const char* e = std::getenv("AMLT_HOST_PANEL_BYTES")) panel_bytes = std::max(1.0, std::atof(e));
        const double b_bytes = double(K) * double(host_ops->b.ld) * es;
        np = static_cast<int>(std::max(1.0, std::min({8.0, std::floor(b_bytes / panel_bytes),
                                                      std::floor(double(K) / 256.0)})));
    }
    // Bands: only the first runs panel by panel, as B arrives; it is tall
    // enough that its compute covers the rest of B's transfer (from the
    // winner's measured seconds per row, assuming ~40 GB/s host copies, more
    // with a broadcast behind them), between 1/8 and 1/2 of the rows. The
    // other bands run whole K (one launch each, no extra R traffic); the last
    // one is an eighth as tall as the others, so the copy-out that trails the
    // final compute is short. 64-row multiples.
    int nb = 1;
    std::vector<int64_t> redge;
    auto layout = [&](bool zero_copy) {
        nb = banded ? static_cast<int>(std::min<int64_t>(8, M / 256)) : 1;
        redge.clear();
        if (nb == 1) {
            redge = {bounds->i0, bounds->i1};
            return;
        }
        const double t_b = double(K) * double(host_ops->b.ld) * es / 40e9 * (bcast ? 1.25 : 1.0);
        const double t_a = double(bytes[0]) / 40e9;
        // band 0's rows: with a measured rate, tall enough that its compute
        // covers B's transfer (K panels) or, zero-copy, B's and all of A's
        // (the later rows then never wait); between M/8 and M/2
        auto rows0_of = [&](int bands) {
            int64_t r = M / bands;
            if (row_seconds > 0.0 && (zero_copy || np > 1))
                r = static_cast<int64_t>(std::ceil(1.3 * (t_b + (zero_copy ? t_a : 0.0)) / row_seconds));
            r = std::min<int64_t>(std::max<int64_t>(r, M / 8), M / 2) / 64 * 64;
            return std::max<int64_t>(r, std::min<int64_t>(M, 64));
        };
        {
            // Band count: every band boundary drains the GPU (up to a wave of
            // CTAs idles), while more bands hide more of the A / R transfers.
            // With the winner's measured seconds per row, minimise boundaries
            // x wave time + exposed copy (~ copy time / bands): nb = sqrt(copy
            // x waves / compute); without it, as many bands as full waves
            // allow. At most 8, at least one wave each (split-K multiplies
            // CTAs). Zero-copy: only A is copied; when band 0's compute covers
            // every copy, or without a measured rate, the other rows run as
            // one launch (at least 2 bands: band 0 is staged).
            const VariantDesc& v = vdesc(vi);
            const int64_t splits = ((!v.run || v.splittable) && split_winner) ? (K + tp.kc - 1) / tp.kc : 1;
            const int64_t slots = int64_t(ctx->num_sms) * occ_of(ctx, vi);
            const int64_t fill = ctas_for(v, M, N) * splits / std::max<int64_t>(1, slots);
            int64_t want = zero_copy ? 2 : fill;
            if (row_seconds > 0.0) {
                const double compute_s = row_seconds * double(M);
                const double copy_s = zero_copy ? t_a : (double(bytes[0]) + double(bytes[2]) * (r_zero ? 1.0 : 2.0)) / 40e9;
                want = static_cast<int64_t>(std::lround(std::sqrt(copy_s * double(std::max<int64_t>(fill, 1)) / compute_s)));
                if (zero_copy && double(rows0_of(2)) * row_seconds >= t_b + t_a) want = 2;
            }
            nb = static_cast<int>(std::max<int64_t>(zero_copy ? 2 : 1, std::min<int64_t>({int64_t(nb), fill, want})));
        }
        if (nb == 1) {
            redge = {bounds->i0, bounds->i1};
            return;
        }
        const int64_t rows0 = rows0_of(nb);
        redge.push_back(bounds->i0);
        const std::vector<int64_t> rest = band_edges(bounds->i0 + rows0, M - rows0, nb - 1, 64, true);
        redge.insert(redge.end(), rest.begin(), rest.end());
    };
    layout(r_mapped != nullptr);
    if (r_mapped) {
        // every zero-copy band must run unpacked, on a variant whose epilogue
        // (and split-K reduce) honours r_zero (else: the staged pipeline)
        amlt_operands probe = hview;
        probe.r.data = r_mapped;
        bool ok = nb >= 2;
        for (int b = 1; ok && b < nb; ++b) {
            amlt_bounds bb = *bounds;
            bb.i0 = redge[static_cast<size_t>(b)];
            bb.i1 = redge[static_cast<size_t>(b) + 1];
            const Resolved rv = resolve(plan, &probe, &bb);
            ok = !rv.packed() && vdesc(plan_dispatch(ctx, plan, &tp, rv).variant).r_overwrite;
        }
        if (!ok) {
            r_mapped = nullptr;
            layout(false);
        }
    }
    const bool zc = r_mapped != nullptr;

    // A of band 0 arrives K panel by K panel with B (a 2-D copy per panel)
    // when its rows are k-contiguous, so compute waits for one panel of each.
    const bool a0_panels = np > 1 && a_rows;
    // Panels: edges on multiples of 64 k (16-byte aligned operand offsets),
    // growing geometrically by g: compute starts after the first (thin)
    // panel's copy, and panel p+1 (g times deeper) still lands before panel
    // p is done as long as band 0 computes a k row at least g times faster
    // than one crosses the bus (rho, from the winner's seconds per row;
    // g = rho, at most 1.5). With a broadcast every rank must cut B the same
    // way whatever its rows or tuning, so the edges depend on K and np only:
    // g = 1.25, which band 0's height (its compute covers 1.3x the copies)
    // sustains.
    std::vector<int64_t> kedge = band_edges(bounds->k0, K, np, 64, false);
    if (np > 1) {
        double g = bcast ? 1.25 : 1.0;
        if (!bcast && row_seconds > 0.0) {
            const double rows0 = double(redge[1] - redge[0]);
            const double comp_k = rows0 * row_seconds / double(K);
            const double xfer_k = (double(host_ops->b.ld) * es + (a0_panels ? rows0 * es : 0.0)) / 40e9;
            g = std::min(1.5, std::max(1.0, comp_k / xfer_k));
        }
        if (g > 1.0) {
            double total = 0.0, w = 1.0;
            for (int p = 0; p < np; ++p, w *= g) total += w;
            std::vector<int64_t> e(1, bounds->k0);
            double cum = 0.0;
            w = 1.0;
            for (int p = 0; p + 1 < np; ++p, w *= g) {
                cum += w;
                int64_t k = static_cast<int64_t>(std::llround(double(K) * cum / total / 64.0)) * 64;
                k = std::max(k, e.back() - bounds->k0 + 64);
                if (k >= K) break;
                e.push_back(bounds->k0 + k);
            }
            e.push_back(bounds->k0 + K);
            if (static_cast<int>(e.size()) == np + 1) kedge = e;  // (else keep equal panels)
        }
    }

    // device staging, one buffer per operand (same pitch and offsets as the
    // host's); with the result going straight to the host, R is staged for
    // band 0's rows only
    amlt_operands dev = hview;
    amlt_matrix* dslot[5 + AMLT_MAX_AUX] = {&dev.a, &dev.b, &dev.r, &dev.thres, &dev.dis};
    for (int q = 0; q + 5 < nslot; ++q) dslot[5 + q] = &dev.aux[q];
    const int64_t arow = host_ops->a.ld * es, rrow = host_ops->r.ld * es;
    for (int s = 0; s < nslot; ++s) {
        if (!hslot[s]->data) continue;
        size_t need = bytes[s];
        if (s == 2 && zc) need = std::min(need, size_t(redge[1]) * size_t(rrow));
        if (!need) {
            dslot[s]->data = ctx->hbuf[s] ? ctx->hbuf[s] : reinterpret_cast<void*>(uintptr_t(256));
            continue;
        }
        if (need > ctx->hbuf_bytes[s]) {
            if (ctx->hbuf[s]) cudaFree(ctx->hbuf[s]);
            ctx->hbuf[s] = nullptr;
            ctx->hbuf_bytes[s] = 0;
            cuda_check(cudaMalloc(&ctx->hbuf[s], need), "cudaMalloc(host staging)");
            ctx->hbuf_bytes[s] = need;
        }
        dslot[s]->data = ctx->hbuf[s];
    }
    amlt_operands dev_zc = dev;  // bands after the first, R in host memory
    if (zc) dev_zc.r.data = r_mapped;
    if (!ctx->copy_in) {
        cuda_check(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking), "cudaStreamCreate");
        cuda_check(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking), "cudaStreamCreate");
    }

    // events: [0] start, [1] replicated operands ready, [2..2+nb) band inputs,
    // [2+nb..2+nb+np) panels ready, [2+nb+np..2+2nb+np) bands done,
    // [2+2nb+np..2+2nb+2np) band 0's A panels, [last] out
    const int nev = 3 + 2 * nb + 2 * np;
    while (static_cast<int>(ctx->pipe_ev.size()) < nev) {
        cudaEvent_t e;
        cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        ctx->pipe_ev.push_back(e);
    }
    cudaEvent_t* ev = ctx->pipe_ev.data();
    cudaEvent_t start_ev = ev[0], small_ev = ev[1], out_ev = ev[nev - 1];
    auto band_in = [&](int b) { return ev[2 + b]; };
    auto panel_ev = [&](int p) { return ev[2 + nb + p]; };
    auto band_done = [&](int b) { return ev[2 + nb + np + b]; };
    auto a0_ev = [&](int p) { return ev[2 + 2 * nb + np + p]; };

    const int64_t brow = host_ops->b.ld * es;  // one k row of B (b_kouter)
    // k rows [k0, k1) of B, relative to the buffer (the bounds' k0 is an offset into it)
    auto b_span = [&](int64_t k0, int64_t k1, size_t* off, size_t* len) {
        if (np == 1) {
            *off = 0;
            *len = bytes[1];
        } else {
            *off = std::min(size_t(k0) * size_t(brow), bytes[1]);
            *len = std::min(size_t(k1 - k0) * size_t(brow), bytes[1] - *off);
        }
    };
    auto h2d = [&](void* dst, const void* src, size_t n, cudaStream_t s, const char* what) {
        if (n) cuda_check(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, s), what);
    };
    auto bcast_bytes = [&](void* buf, size_t n) {
        if (n) nccl_check(nccl().bcast(buf, buf, n, kNcclUint8, 0, ctx->comm, ctx->comm_stream), "ncclBroadcast");
    };
    // band b's A rows (unless they come panel by panel) and R rows (staged
    // bands only: zeroed, or copied in)
    auto copy_band_in = [&](int b) {
        const int64_t r0 = redge[static_cast<size_t>(b)], r1 = redge[static_cast<size_t>(b) + 1];
        const bool with_a = !(b == 0 && a0_panels);
        const bool with_r = !(zc && b > 0);
        if (nb == 1) {
            if (with_a) h2d(ctx->hbuf[0], host_ops->a.data, bytes[0], ctx->copy_in, "H2D A");
            if (r_zero) cuda_check(cudaMemsetAsync(ctx->hbuf[2], 0, bytes[2], ctx->copy_in), "memset R");
            else h2d(ctx->hbuf[2], host_ops->r.data, bytes[2], ctx->copy_in, "H2D R");
        } else {
            if (with_r) {
                if (r_zero)
                    cuda_check(cudaMemsetAsync(static_cast<char*>(ctx->hbuf[2]) + r0 * rrow, 0, size_t(r1 - r0) * rrow,
                                               ctx->copy_in), "memset R band");
                else
                    h2d(static_cast<char*>(ctx->hbuf[2]) + r0 * rrow,
                        static_cast<const char*>(host_ops->r.data) + r0 * rrow, size_t(r1 - r0) * rrow, ctx->copy_in,
                        "H2D R band");
            }
            if (with_a)
                h2d(static_cast<char*>(ctx->hbuf[0]) + r0 * arow, static_cast<const char*>(host_ops->a.data) + r0 * arow,
                    size_t(r1 - r0) * arow, ctx->copy_in, "H2D A band");
        }
        cuda_check(cudaEventRecord(band_in(b), ctx->copy_in), "cudaEventRecord");
    };
    auto copy_panel_in = [&](int p) {
        const int64_t k0 = kedge[static_cast<size_t>(p)], k1 = kedge[static_cast<size_t>(p) + 1];
        if (a0_panels) {  // band 0's A, k columns [k0, k1)
            const size_t off = size_t(redge[0]) * size_t(arow) + size_t(k0) * es;
            if (k1 > k0 && redge[1] > redge[0])
                cuda_check(cudaMemcpy2DAsync(static_cast<char*>(ctx->hbuf[0]) + off, size_t(arow),
                                             static_cast<const char*>(host_ops->a.data) + off, size_t(arow),
                                             size_t(k1 - k0) * es, size_t(redge[1] - redge[0]),
                                             cudaMemcpyHostToDevice, ctx->copy_in),
                           "H2D A panel");
            cuda_check(cudaEventRecord(a0_ev(p), ctx->copy_in), "cudaEventRecord");
        }
        size_t off, len;
        b_span(k0, k1, &off, &len);
        if (root) h2d(static_cast<char*>(ctx->hbuf[1]) + off, static_cast<const char*>(host_ops->b.data) + off, len,
                      ctx->copy_in, "H2D B panel");
        if (bcast) {
            if (root) {
                cuda_check(cudaEventRecord(panel_ev(p), ctx->copy_in), "cudaEventRecord");
                cuda_check(cudaStreamWaitEvent(ctx->comm_stream, panel_ev(p), 0), "cudaStreamWaitEvent");
            }
            bcast_bytes(static_cast<char*>(ctx->hbuf[1]) + off, len);
            cuda_check(cudaEventRecord(panel_ev(p), ctx->comm_stream), "cudaEventRecord");
        } else {
            cuda_check(cudaEventRecord(panel_ev(p), ctx->copy_in), "cudaEventRecord");
        }
    };
    auto band_bounds = [&](int b, int p) {
        amlt_bounds bb = *bounds;
        bb.i0 = redge[static_cast<size_t>(b)];
        bb.i1 = redge[static_cast<size_t>(b) + 1];
        bb.k0 = kedge[static_cast<size_t>(p)];
        bb.k1 = kedge[static_cast<size_t>(p) + 1];
        return bb;
    };

    // AMLT_HOST_TRACE=1: timing events at the stage boundaries, printed to
    // stderr after the call (pipeline diagnostics; off by default)
    const bool trace = std::getenv("AMLT_HOST_TRACE") != nullptr;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    auto mark = [&](const std::string& what, cudaStream_t s) {
        if (!trace) return;
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "cudaEventCreate");
        cuda_check(cudaEventRecord(e, s), "cudaEventRecord");
        marks.emplace_back(what, e);
    };
    auto body = [&] {
        cuda_check(cudaEventRecord(start_ev, ctx->stream), "cudaEventRecord");
        mark("start", ctx->stream);
        cuda_check(cudaStreamWaitEvent(ctx->copy_in, start_ev, 0), "cudaStreamWaitEvent");
        if (bcast) cuda_check(cudaStreamWaitEvent(ctx->comm_stream, start_ev, 0), "cudaStreamWaitEvent");
        // replicated operands other than B (thresholds, vectors, [i] / [i][j]
        // leaves are copied whole by every rank: they are the rank's own)
        for (int s = 3; s < nslot; ++s)
            if (bytes[s] && (root || !shared[static_cast<size_t>(s)]))
                h2d(ctx->hbuf[s], hslot[s]->data, bytes[s], ctx->copy_in, "H2D operand");
        cuda_check(cudaEventRecord(small_ev, ctx->copy_in), "cudaEventRecord");
        if (bcast) {
            cuda_check(cudaStreamWaitEvent(ctx->comm_stream, small_ev, 0), "cudaStreamWaitEvent");
            nccl_check(nccl().group_start(), "ncclGroupStart");
            for (int s = 3; s < nslot; ++s)
                if (bytes[s] && shared[static_cast<size_t>(s)]) bcast_bytes(ctx->hbuf[s], bytes[s]);
            nccl_check(nccl().group_end(), "ncclGroupEnd");
            cuda_check(cudaEventRecord(small_ev, ctx->comm_stream), "cudaEventRecord");
        }
        cuda_check(cudaStreamWaitEvent(ctx->stream, small_ev, 0), "cudaStreamWaitEvent");
        // inputs: band 0 (R, and A unless it comes with the panels), the B
        // panels (band 0 consumes them as they land), then the other A bands
        copy_band_in(0);
        mark("band 0 in", ctx->copy_in);
        copy_panel_in(0);
        mark("panel 0 in", bcast ? ctx->comm_stream : ctx->copy_in);
        for (int p = 1; p < np; ++p) copy_panel_in(p);
        mark("panels in", bcast ? ctx->comm_stream : ctx->copy_in);
        for (int b = 1; b < nb; ++b) copy_band_in(b);
        mark("bands in", ctx->copy_in);
        if (tune_now) {
            for (int b = 0; b < nb; ++b) cuda_check(cudaStreamWaitEvent(ctx->stream, band_in(b), 0), "cudaStreamWaitEvent");
            for (int p = 0; p < np; ++p) {
                cuda_check(cudaStreamWaitEvent(ctx->stream, panel_ev(p), 0), "cudaStreamWaitEvent");
                if (a0_panels) cuda_check(cudaStreamWaitEvent(ctx->stream, a0_ev(p), 0), "cudaStreamWaitEvent");
            }
            adaptive(ctx, plan, &dev, *bounds, clock, clock_user, nullptr, rep);
            cuda_check(cudaEventRecord(band_done(0), ctx->stream), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(ctx->copy_out, band_done(0), 0), "cudaStreamWaitEvent");
            cuda_check(cudaMemcpyAsync(host_ops->r.data, ctx->hbuf[2], bytes[2], cudaMemcpyDeviceToHost,
                                       ctx->copy_out), "D2H R");
        } else {
            for (int b = 0; b < nb; ++b) {
                cuda_check(cudaStreamWaitEvent(ctx->stream, band_in(b), 0), "cudaStreamWaitEvent");
                // band 0 panel by panel as B lands; the others whole K
                const int parts = b == 0 ? np : 1;
                amlt_bounds bb{};
                KParams whole_k{};  // band 0's preparation of B, as one whole-K preparation
                const VariantDesc* prepped = nullptr;
                for (int p = 0; p < parts; ++p) {
                    bb = band_bounds(b, p);
                    if (b > 0) {
                        bb.k0 = bounds->k0;
                        bb.k1 = bounds->k1;
                    } else {
                        cuda_check(cudaStreamWaitEvent(ctx->stream, panel_ev(p), 0), "cudaStreamWaitEvent");
                        if (a0_panels) cuda_check(cudaStreamWaitEvent(ctx->stream, a0_ev(p), 0), "cudaStreamWaitEvent");
                    }
                    if (b == 0 && p == 0) mark("compute begins", ctx->stream);
                    const bool to_host = zc && b > 0;
                    Resolved rv = resolve(plan, to_host ? &dev_zc : &dev, &bb);
                    if (to_host) rv.kp.r_zero = r_zero ? 1 : 0;
                    Dispatch dp = plan_dispatch(ctx, plan, &tp, rv);
                    const VariantDesc& v = vdesc(dp.variant);
                    if (b == 0 && np > 1 && d.accumulate && v.run && v.prep_b && v.prep_panels && !rv.packed() &&
                        rv.M > 0 && rv.N > 0 && rv.K > 0) {
                        // B prepared panel by panel into one whole-K
                        // preparation, which the later bands reuse as is
                        rv.kp.plane_k0 = bb.k0 - bounds->k0;
                        rv.kp.plane_kdim = K;
                        ensure_tc_ws(ctx, v, rv.kp);
                        cuda_check(v.prep_b(rv.kp, ctx->tc_ws, ctx->stream), "B preparation (panel)");
                        bprep_mark(ctx, v, rv.kp);
                        if (p == 0) {
                            whole_k = rv.kp;
                            whole_k.K = K;
                            prepped = &v;
                        }
                    }
                    enqueue(ctx, plan, rv, dp);
                }
                if (prepped) bprep_mark(ctx, *prepped, whole_k);
                if (b == 0)  // (every panel has landed once band 0 is done)
                    for (int p = 0; p < np; ++p)
                        cuda_check(cudaStreamWaitEvent(ctx->stream, panel_ev(p), 0), "cudaStreamWaitEvent");
                mark("band " + std::to_string(b) + " computed", ctx->stream);
                cuda_check(cudaEventRecord(band_done(b), ctx->stream), "cudaEventRecord");
                if (zc && b > 0) continue;  // its rows are in host memory already
                cuda_check(cudaStreamWaitEvent(ctx->copy_out, band_done(b), 0), "cudaStreamWaitEvent");
                const int64_t r0 = bb.i0, r1 = bb.i1;
                if (nb == 1)
                    cuda_check(cudaMemcpyAsync(host_ops->r.data, ctx->hbuf[2], bytes[2], cudaMemcpyDeviceToHost,
                                               ctx->copy_out), "D2H R");
                else
                    cuda_check(cudaMemcpyAsync(static_cast<char*>(host_ops->r.data) + r0 * rrow,
                                               static_cast<const char*>(ctx->hbuf[2]) + r0 * rrow,
                                               size_t(r1 - r0) * rrow, cudaMemcpyDeviceToHost, ctx->copy_out),
                               "D2H R band");
            }
        }
        mark("R out", ctx->copy_out);
        cuda_check(cudaEventRecord(out_ev, ctx->copy_out), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(ctx->stream, out_ev, 0), "cudaStreamWaitEvent");
        if (bcast) {  // the comm stream's work is part of this call
            cuda_check(cudaEventRecord(small_ev, ctx->comm_stream), "cudaEventRecord");
            cuda_check(cudaStreamWaitEvent(ctx->stream, small_ev, 0), "cudaStreamWaitEvent");
        }
    };
    double el = 0;
    if (clock && !tune_now) {
        const double t0 = clock(clock_user);
        body();
        cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
        el = clock(clock_user) - t0;
    } else {
        // (tuning with a caller clock: the tuner reads it around each of its
        // subtasks, as adaptive_execute does; the call is timed by events)
        // (own timing events: the tuner's trials use ev0 / ev1)
        if (!ctx->hev0) {
            cuda_check(cudaEventCreate(&ctx->hev0), "cudaEventCreate");
            cuda_check(cudaEventCreate(&ctx->hev1), "cudaEventCreate");
        }
        cuda_check(cudaEventRecord(ctx->hev0, ctx->stream), "cudaEventRecord");
        body();
        cuda_check(cudaEventRecord(ctx->hev1, ctx->stream), "cudaEventRecord");
        cuda_check(cudaEventSynchronize(ctx->hev1), "cudaEventSynchronize");
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, ctx->hev0, ctx->hev1), "cudaEventElapsedTime");
        el = ms * 1e-3;
        if (tune_now && clock) el = rep->total_seconds;
    }
    if (trace && !marks.empty()) {
        cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
        std::fprintf(stderr, "[amlt host pipeline] nb=%d np=%d M=%lld N=%lld K=%lld bcast=%d zero-copy R=%d "
                             "rows0=%lld k-panel0=%lld\n", nb, np, (long long)M, (long long)N, (long long)K,
                     bcast ? 1 : 0, zc ? 1 : 0, (long long)(redge[1] - redge[0]), (long long)(kedge[1] - kedge[0]));
        for (auto& m : marks) {
            float ms = 0;
            cudaEventElapsedTime(&ms, marks.front().second, m.second);
            std::fprintf(stderr, "[amlt host pipeline]   %8.2f ms  %s\n", ms, m.first.c_str());
        }
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
    {
        int64_t* L = ctx->host_layout;
        L[0] = nb;
        L[1] = np;
        L[2] = zc ? 1 : 0;
        L[3] = redge[1] - redge[0];
        L[4] = kedge[1] - kedge[0];
        L[5] = bcast ? 1 : 0;
        L[6] = tune_now ? 1 : 0;
    }
    if (rep && !tune_now) {
        std::memset(rep, 0, sizeof(*rep));
        rep->best_variant = plan_local_index(plan, vi);
        rep->best_kc = split_winner ? tp.kc : K;
        rep->from_cache = cached ? 1 : 0;
        // completed regions: band 0 per K panel, the other bands whole K
        for (int p = 0; p < np; ++p)
            add_cover(rep, amlt_bounds{redge[0], redge[1], bounds->j0, bounds->j1, kedge[static_cast<size_t>(p)],
                                       kedge[static_cast<size_t>(p) + 1]});
        for (int b = 1; b < nb; ++b)
            add_cover(rep, amlt_bounds{redge[static_cast<size_t>(b)], redge[static_cast<size_t>(b) + 1], bounds->j0,
                                       bounds->j1, bounds->k0, bounds->k1});
        rep->total_seconds = el;
    } else if (rep && tune_now) {
        // the report's subtasks plus the copies around them
        if (!clock) rep->total_seconds = el;
        // a later call of this shape reuses the winner
    }
    if (elapsed_s) *elapsed_s = el;
}

// ---------------------------------------------------------------------------
// boundary helpers

template <class F>
amlt_status guarded(amlt_ctx* ctx, F&& f) {
    if (ctx) ++ctx->call_gen;  // operand preparations do not outlive the call
    try {
        f();
        if (ctx && !ctx->dry()) {
            // no CUDA error may outlive the call that caused it
            const cudaError_t pend = cudaPeekAtLastError();
            if (pend != cudaSuccess)
                throw EngineError(AMLT_ERR_CUDA, std::string("CUDA error left by this call: ") +
                                                     cudaGetErrorString(pend));
        }
        if (ctx) ctx->err.clear();
        return AMLT_OK;
    } catch (const EngineError& e) {
        if (ctx) ctx->err = e.what();
        else g_create_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        if (ctx) ctx->err = e.what();
        else g_create_error = e.what();
        return AMLT_ERR_ENGINE;
    }
}

}  // namespace

namespace amltk {
// A rank of a single-process group (csrc/sharded.cu) uses a communicator the
// group owns (ncclCommInitAll).
amlt_status ctx_use_comm(amlt_ctx* ctx, void* comm, int rank, int nranks) {
    if (!ctx) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        comm_use(ctx, static_cast<ncclComm_t>(comm), rank, nranks, false);
    });
}
}  // namespace amltk

// ===========================================================================
// C ABI

extern "C" {

int amlt_gpu_abi_version(void) { return AMLT_GPU_ABI_VERSION; }

const char* amlt_gpu_last_error(const amlt_ctx* ctx) {
    return ctx ? ctx->err.c_str() : g_create_error.c_str();
}

amlt_status amlt_gpu_ctx_create(int device, int flags, amlt_ctx** out) {
    if (!out) return AMLT_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    amlt_ctx* ctx = new amlt_ctx();
    ctx->device = device;
    ctx->flags = flags;
    const auto& reg = registry();
    std::lock_guard<std::mutex> reg_lock(registry_mutex());  // a consistent snapshot of the registry
    amlt_status st = guarded(nullptr, [&] {
        if (ctx->dry()) {
            ctx->occupancy.assign(reg.variants.size(), 0);
            for (size_t i = 0; i < reg.variants.size(); ++i) ctx->occupancy[i] = reg.variants[i].minb;
            return;
        }
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            fail(AMLT_ERR_NO_DEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
        if (device < 0 || device >= n) fail(AMLT_ERR_NO_DEVICE, "device index out of range");
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10 || prop.minor != 0)
            fail(AMLT_ERR_NO_DEVICE, std::string("device is sm_") + std::to_string(prop.major) +
                                         std::to_string(prop.minor) +
                                         "; this build targets sm_100a (B200) only");
        ctx->num_sms = prop.multiProcessorCount;
        // The context's own stream is a BLOCKING stream: it is ordered with
        // the legacy default stream, where callers without a stream of their
        // own (PyTorch's default) produce the operands. (A non-blocking one
        // let a kernel start before the caller's zero-fill of R had run.)
        cuda_check(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamDefault), "cudaStreamCreate");
        ctx->stream = ctx->own_stream;
        cuda_check(cudaEventCreate(&ctx->ev0), "cudaEventCreate");
        cuda_check(cudaEventCreate(&ctx->ev1), "cudaEventCreate");
        // Load every kernel now (lazy module loading would otherwise charge
        // the first tuning trial) and size its occupancy.
        ctx->occupancy.assign(reg.variants.size(), 1);
        for (size_t i = 0; i < reg.variants.size(); ++i) {
            const VariantDesc& v = reg.variants[i];
            if (!v.launch) {  // run-time compiled: loaded and sized on demand
                ctx->occupancy[i] = 0;
                continue;
            }
            cuda_check(cudaFuncSetAttribute(v.func, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem),
                       "cudaFuncSetAttribute");
            int occ = 0;
            cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, v.func, v.threads, v.smem),
                       "cudaOccupancyMaxActiveBlocksPerMultiprocessor");
            if (occ < 1) fail(AMLT_ERR_NO_FEASIBLE_KERNEL, std::string("variant ") + v.name + " cannot be resident");
            ctx->occupancy[i] = occ;
        }
        for (const auto& a : reg.aux) {
            if (!a.assign) continue;  // run-time compiled body
            cudaFuncAttributes fa;
            cuda_check(cudaFuncGetAttributes(&fa, a.assign_func), "cudaFuncGetAttributes");
            cuda_check(cudaFuncGetAttributes(&fa, a.reduce_func), "cudaFuncGetAttributes");
            cuda_check(cudaFuncGetAttributes(&fa, a.pack_func), "cudaFuncGetAttributes");
        }
    });
    if (st != AMLT_OK) {
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
        delete ctx;
        return st;
    }
    *out = ctx;
    return AMLT_OK;
}

void amlt_gpu_ctx_destroy(amlt_ctx* ctx) {
    if (!ctx) return;
    if (!ctx->dry()) {
        cudaSetDevice(ctx->device);
        if (ctx->own_stream) cudaStreamSynchronize(ctx->own_stream);
        if (ctx->comm_stream) cudaStreamSynchronize(ctx->comm_stream);
        comm_release(ctx);
        if (ctx->work) cudaFree(ctx->work);
        if (ctx->pack_ws) cudaFree(ctx->pack_ws);
        if (ctx->scratch) cudaFree(ctx->scratch);
        if (ctx->tc_ws) cudaFree(ctx->tc_ws);
        for (void* p : ctx->hbuf)
            if (p) cudaFree(p);
        if (ctx->ev0) cudaEventDestroy(ctx->ev0);
        if (ctx->ev1) cudaEventDestroy(ctx->ev1);
        if (ctx->hev0) cudaEventDestroy(ctx->hev0);
        if (ctx->hev1) cudaEventDestroy(ctx->hev1);
        if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
        for (cudaEvent_t e : ctx->pipe_ev) cudaEventDestroy(e);
        if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
        if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
        if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    }
    delete ctx;
}

amlt_status amlt_gpu_set_stream(amlt_ctx* ctx, void* stream) {
    if (!ctx) return AMLT_ERR_INVALID_ARGUMENT;
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return AMLT_OK;
}

void amlt_gpu_clear_tuning_cache(amlt_ctx* ctx) {
    if (ctx) ctx->tune_cache.clear();
}

amlt_status amlt_gpu_plan_create(amlt_ctx* ctx, const amlt_body_desc* desc, amlt_plan** out) {
    if (!ctx || !desc || !out) return AMLT_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    amlt_plan* plan = new amlt_plan();
    amlt_status st = guarded(ctx, [&] {
        const amlt_body_desc& d = *desc;
        if (d.body == AMLT_BODY_GENERIC)
            fail(AMLT_ERR_UNSUPPORTED,
                 "generated bodies are planned from the task text (amlt_gpu_plan_from_source)");
        if (d.body < AMLT_BODY_GEMM || d.body > AMLT_BODY_THRCOUNT)
            fail(AMLT_ERR_UNSUPPORTED, "unknown body " + std::to_string(d.body));
        if (d.dtype < AMLT_F64 || d.dtype > AMLT_I32)
            fail(AMLT_ERR_INVALID_ARGUMENT, "unknown dtype " + std::to_string(d.dtype));
        if ((d.layout_a != AMLT_LAYOUT_NORMAL && d.layout_a != AMLT_LAYOUT_TRANSPOSED) ||
            (d.layout_b != AMLT_LAYOUT_NORMAL && d.layout_b != AMLT_LAYOUT_TRANSPOSED))
            fail(AMLT_ERR_INVALID_ARGUMENT, "unknown operand layout");
        const bool needs_t = d.body == AMLT_BODY_DISCOUNT || d.body == AMLT_BODY_BOOST ||
                             d.body == AMLT_BODY_THRCOUNT;
        if (d.thres_class < AMLT_LEAF_CONSTANT || d.thres_class > AMLT_LEAF_MAT_IJ)
            fail(AMLT_ERR_INVALID_ARGUMENT, "unknown threshold leaf class");
        // thresholds indexed by i or (i, j) run the per-output-threshold variants
        const bool tout =
            needs_t && (d.thres_class == AMLT_LEAF_VEC_I || d.thres_class == AMLT_LEAF_MAT_IJ);
        plan->desc = d;
        plan->ctx = ctx;
        plan->aux = find_aux(d.body, d.dtype);
        if (!plan->aux)
            fail(AMLT_ERR_UNSUPPORTED, std::string("no GPU kernel for body ") + body_name(d.body) +
                                           " in " + dtype_name(d.dtype));
        const auto& reg = registry();
        std::lock_guard<std::mutex> reg_lock(registry_mutex());
        for (size_t i = 0; i < reg.variants.size(); ++i)
            if (reg.variants[i].body == d.body && reg.variants[i].dtype == d.dtype &&
                reg.variants[i].tout == tout)
                plan->variants.push_back(static_cast<int>(i));
        if (plan->variants.empty())
            fail(AMLT_ERR_NO_FEASIBLE_KERNEL, "no tile variant compiled for this body/dtype");
    });
    if (st != AMLT_OK) {
        delete plan;
        return st;
    }
    *out = plan;
    return AMLT_OK;
}

amlt_status amlt_gpu_recognize(const char* task_source, amlt_task_info* info) {
    if (!task_source || !info) return AMLT_ERR_INVALID_ARGUMENT;
    try {
        amltk::RecognizedTask rt = amltk::recognize_task(task_source);
        std::memset(info, 0, sizeof(*info));
        info->desc = rt.desc;
        auto put = [](char* dst, const std::string& s) {
            std::snprintf(dst, 64, "%s", s.c_str());
        };
        put(info->a, rt.a);
        put(info->b, rt.b);
        put(info->r, rt.r);
        put(info->thres, rt.thres);
        put(info->dis, rt.dis);
        for (int c = 0; c < AMLT_PROG_NOPS; ++c) info->prog_counts[c] = rt.prog_counts[c];
        info->prog_instrs = rt.prog_instrs;
        info->prog_flops = rt.prog_flops;
        info->n_aux = static_cast<int32_t>(rt.aux_names.size());
        for (size_t q = 0; q < rt.aux_names.size(); ++q) {
            put(info->aux_names[q], rt.aux_names[q]);
            info->aux_class[q] = rt.aux_class[q];
        }
        g_create_error.clear();
        return AMLT_OK;
    } catch (const amltk::TaskError& e) {
        g_create_error = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_create_error = e.what();
        return AMLT_ERR_ENGINE;
    }
}

amlt_status amlt_gpu_plan_from_source(amlt_ctx* ctx, const char* task_source, int dtype,
                                      amlt_plan** out, amlt_task_info* info) {
    if (!ctx || !out) return AMLT_ERR_INVALID_ARGUMENT;
    amlt_task_info local;
    amlt_task_info* ti = info ? info : &local;
    amlt_status st = amlt_gpu_recognize(task_source, ti);
    if (st != AMLT_OK) {
        ctx->err = g_create_error;
        return st;
    }
    ti->desc.dtype = dtype;
    if (ti->desc.body != AMLT_BODY_GENERIC) return amlt_gpu_plan_create(ctx, &ti->desc, out);
    *out = nullptr;
    amlt_plan* plan = new amlt_plan();
    st = guarded(ctx, [&] {
        if (dtype != AMLT_F64 && dtype != AMLT_F32)
            fail(AMLT_ERR_UNSUPPORTED, "generated bodies compute in f64 or f32");
        amltk::RecognizedTask rt;
        try {
            rt = amltk::recognize_task(task_source);
            const amltk::JitBody& jb = amltk::jit_body(rt, dtype, !ctx->dry());
            plan->variants = jb.variants;
            plan->aux = jb.aux;
        } catch (const amltk::TaskError& e) {
            fail(e.code, e.what());
        }
        plan->desc = ti->desc;
        plan->ctx = ctx;
        plan->aux_names = rt.aux_names;
        plan->aux_class = rt.aux_class;
    });
    if (st != AMLT_OK) {
        delete plan;
        return st;
    }
    *out = plan;
    return AMLT_OK;
}

int64_t amlt_gpu_generated_source(const char* task_source, int dtype, char* buf, int64_t buflen) {
    if (!task_source) return -1;
    try {
        amltk::RecognizedTask rt = amltk::recognize_task(task_source);
        if (rt.desc.body != AMLT_BODY_GENERIC) {
            g_create_error = "statement has a fixed body; no generated source";
            return -1;
        }
        const std::string src = amltk::jit_source(rt, dtype);
        if (buf && buflen > 0) std::snprintf(buf, static_cast<size_t>(buflen), "%s", src.c_str());
        return static_cast<int64_t>(src.size());
    } catch (const std::exception& e) {
        g_create_error = e.what();
        return -1;
    }
}

void amlt_gpu_plan_destroy(amlt_plan* plan) { delete plan; }

int amlt_gpu_plan_num_variants(const amlt_plan* plan) {
    return plan ? static_cast<int>(plan->variants.size()) : 0;
}

amlt_status amlt_gpu_plan_variant(const amlt_plan* plan, int idx, amlt_variant_info* info) {
    if (!plan || !info || idx < 0 || idx >= (int)plan->variants.size()) return AMLT_ERR_INVALID_ARGUMENT;
    const VariantDesc& v = vdesc(plan->variants[static_cast<size_t>(idx)]);
    std::memset(info, 0, sizeof(*info));
    info->index = idx;
    info->body = v.body;
    info->dtype = v.dtype;
    info->block_m = v.bm;
    info->block_n = v.bn;
    info->block_k = v.bk;
    info->thread_m = v.tm;
    info->thread_n = v.tn;
    info->threads = v.threads;
    info->stages = v.stages;
    info->smem_bytes = v.smem;
    info->tensor_core = v.tc ? 1 : 0;
    std::snprintf(info->name, sizeof(info->name), "%s_%s_%dx%d_%s", body_name(v.body),
                  dtype_name(v.dtype), v.bm, v.bn, v.name);
    return AMLT_OK;
}

int amlt_gpu_plan_default_variant(const amlt_plan* plan, int64_t M, int64_t N, int64_t K) {
    (void)K;
    if (!plan) return -1;
    try {
        return plan_local_index(plan, default_variant(plan->ctx, plan, M, N, true));
    } catch (...) {
        return -1;
    }
}

amlt_status amlt_gpu_run_subtask(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                                 const amlt_tile_params* tile, const amlt_bounds* bounds,
                                 amlt_clock_fn clock, void* clock_user, amlt_exec_log* log,
                                 double* elapsed_s) {
    if (!ctx || !plan) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!ctx->dry()) cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        Resolved rv = resolve(plan, ops, bounds);
        Dispatch dp = plan_dispatch(ctx, plan, tile, rv);
        double el = timed_subtask(ctx, plan, rv, dp, *bounds, clock, clock_user, log);
        if (elapsed_s) *elapsed_s = el;
    });
}

amlt_status amlt_gpu_run_naive(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                               const amlt_bounds* bounds, amlt_clock_fn clock, void* clock_user,
                               double* elapsed_s) {
    if (!ctx || !plan) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        // same operand rules as the tiled path; the per-element kernel then
        // addresses every operand through its own strides (no packing)
        Resolved rv = resolve(plan, ops, bounds);
        const amlt_body_desc& d = plan->desc;
        NaiveParams np{};
        char *pa, *pb, *pr;
        stmt_addr(ops->a, d.layout_a, bounds->i0, bounds->k0, "A", &pa, &np.sai, &np.sak);
        stmt_addr(ops->b, d.layout_b, bounds->k0, bounds->j0, "B", &pb, &np.sbk, &np.sbj);
        stmt_addr(ops->r, AMLT_LAYOUT_NORMAL, bounds->i0, bounds->j0, "R", &pr, &np.sri, &np.srj);
        np.A = pa;
        np.B = pb;
        np.R = pr;
        np.thres = rv.kp.thres;
        np.t_si = rv.kp.t_si;
        np.t_sj = rv.kp.t_sj;
        np.tconst = rv.kp.tconst;
        np.dis = rv.kp.dis;
        np.d_sj = rv.kp.d_sj;
        np.M = rv.M;
        np.N = rv.N;
        np.K = rv.K;
        np.accumulate = d.accumulate;
        double el = 0.0;
        if (!ctx->dry()) {
            cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
            const double t0 = clock ? clock(clock_user) : 0.0;
            if (!clock) cuda_check(cudaEventRecord(ctx->ev0, ctx->stream), "cudaEventRecord");
            if (d.body == AMLT_BODY_GENERIC) {
                KParams kp = rv.kp;
                kp.A = np.A;
                kp.B = np.B;
                kp.R = np.R;
                NaiveStrides ns{np.sai, np.sak, np.sbk, np.sbj, np.sri, np.srj, d.accumulate};
                const int64_t total = rv.M * rv.N;
                if (total > 0) {
                    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, int64_t(ctx->num_sms) * 16));
                    void* args[2] = {&kp, &ns};
                    cuda_check(cudaLaunchKernel(plan->aux->naive_func, dim3(blocks), dim3(256), args, 0,
                                                ctx->stream),
                               "naive kernel");
                }
            } else {
                cuda_check(launch_naive(np, d.body, d.dtype, ctx->num_sms, ctx->stream), "naive kernel");
            }
            if (clock) {
                cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
                el = clock(clock_user) - t0;
            } else {
                cuda_check(cudaEventRecord(ctx->ev1, ctx->stream), "cudaEventRecord");
                cuda_check(cudaEventSynchronize(ctx->ev1), "cudaEventSynchronize");
                float ms = 0.f;
                cuda_check(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1), "cudaEventElapsedTime");
                el = ms * 1e-3;
            }
        }
        if (elapsed_s) *elapsed_s = el;
    });
}

amlt_status amlt_gpu_enqueue(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                             const amlt_tile_params* tile, const amlt_bounds* bounds) {
    if (!ctx || !plan) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        Resolved rv = resolve(plan, ops, bounds);
        Dispatch dp = plan_dispatch(ctx, plan, tile, rv);
        enqueue(ctx, plan, rv, dp);
    });
}

struct amlt_graph {
    amlt_ctx* ctx = nullptr;
    cudaGraphExec_t exec = nullptr;
    // the workspaces baked into the graph's kernel parameters
    void* work = nullptr;
    void* tc_ws = nullptr;
    void* pack_ws = nullptr;
};

amlt_status amlt_gpu_graph_capture(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* ops,
                                   const amlt_tile_params* tile, const amlt_bounds* bounds,
                                   amlt_graph** out) {
    if (!ctx || !plan || !out) return AMLT_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    return guarded(ctx, [&] {
        if (ctx->dry()) fail(AMLT_ERR_NO_DEVICE, "amlt_gpu_graph_capture needs a device context");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        Resolved rv = resolve(plan, ops, bounds);
        Dispatch dp = plan_dispatch(ctx, plan, tile, rv);
        // one plain step first: every workspace the step needs is allocated
        // (no allocation may happen inside the capture)
        enqueue(ctx, plan, rv, dp);
        cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
        ++ctx->call_gen;  // the captured step prepares its own B, as every enqueue does
        cudaGraph_t graph = nullptr;
        cuda_check(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal),
                   "cudaStreamBeginCapture");
        try {
            enqueue(ctx, plan, rv, dp);
        } catch (...) {
            cudaGraph_t g = nullptr;
            (void)cudaStreamEndCapture(ctx->stream, &g);
            if (g) cudaGraphDestroy(g);
            (void)cudaGetLastError();
            throw;
        }
        cuda_check(cudaStreamEndCapture(ctx->stream, &graph), "cudaStreamEndCapture");
        cudaGraphExec_t exec = nullptr;
        const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        cuda_check(e, "cudaGraphInstantiate");
        auto* g = new amlt_graph;
        g->ctx = ctx;
        g->exec = exec;
        g->work = ctx->work;
        g->tc_ws = ctx->tc_ws;
        g->pack_ws = ctx->pack_ws;
        *out = g;
    });
}

amlt_status amlt_gpu_graph_launch(amlt_graph* g) {
    if (!g || !g->ctx) return AMLT_ERR_INVALID_ARGUMENT;
    amlt_ctx* ctx = g->ctx;
    return guarded(ctx, [&] {
        if (ctx->work != g->work || ctx->tc_ws != g->tc_ws || ctx->pack_ws != g->pack_ws)
            fail(AMLT_ERR_INVALID_ARGUMENT,
                 "graph invalidated: the context's workspaces were reallocated after the capture");
        cuda_check(cudaGraphLaunch(g->exec, ctx->stream), "cudaGraphLaunch");
    });
}

void amlt_gpu_graph_destroy(amlt_graph* g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    delete g;
}

amlt_status amlt_gpu_adaptive_execute(amlt_ctx* ctx, const amlt_plan* plan,
                                      const amlt_operands* ops, const amlt_bounds* bounds,
                                      int pack, amlt_clock_fn clock, void* clock_user,
                                      amlt_exec_log* log, amlt_tune_report* report) {
    (void)pack;
    if (!ctx || !plan || !bounds) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!ctx->dry()) cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        amlt_tune_report local;
        adaptive(ctx, plan, ops, *bounds, clock, clock_user, log, report ? report : &local);
    });
}

amlt_status amlt_gpu_adaptive_execute_amulet(amlt_ctx* ctx, const amlt_plan* plan,
                                             const amlt_operands* ops, const amlt_bounds* bounds,
                                             int i_h, int i_w, amlt_clock_fn clock,
                                             void* clock_user, amlt_exec_log* log,
                                             amlt_amulet_report* report) {
    if (!ctx || !plan || !bounds || !report || i_h < 1 || i_w < 1) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (!ctx->dry()) cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        std::memset(report, 0, sizeof(*report));
        (void)resolve(plan, ops, bounds);  // validate once up front
        AmuletTuner t{ctx, plan, ops, clock, clock_user, log, report};
        t.run(*bounds, i_h, i_w);
    });
}

amlt_status amlt_gpu_run_host(amlt_ctx* ctx, const amlt_plan* plan, const amlt_operands* host_ops,
                              const amlt_tile_params* tile, const amlt_bounds* bounds, int flags,
                              amlt_clock_fn clock, void* clock_user, double* elapsed_s) {
    if (!ctx || !plan || !host_ops || !bounds) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        host_pipeline(ctx, plan, host_ops, tile, bounds, flags, clock, clock_user, nullptr, elapsed_s);
    });
}

amlt_status amlt_gpu_run_host_adaptive(amlt_ctx* ctx, const amlt_plan* plan,
                                       const amlt_operands* host_ops, const amlt_bounds* bounds,
                                       int flags, amlt_clock_fn clock, void* clock_user,
                                       amlt_tune_report* report, double* elapsed_s) {
    if (!ctx || !plan || !host_ops || !bounds || !report) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        host_pipeline(ctx, plan, host_ops, nullptr, bounds, flags, clock, clock_user, report, elapsed_s);
    });
}

amlt_status amlt_gpu_comm_unique_id(void* id_out) {
    if (!id_out) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(nullptr, [&] {
        if (!nccl().ok) fail(AMLT_ERR_CUDA, "libnccl.so.2 could not be loaded");
        NcclUniqueId id;
        const int r = nccl().get_unique_id(&id);
        if (r != kNcclSuccess) fail(AMLT_ERR_CUDA, std::string("ncclGetUniqueId: ") + nccl_error_string(r));
        std::memcpy(id_out, id.internal, sizeof(id.internal));
    });
}

amlt_status amlt_gpu_comm_attach(amlt_ctx* ctx, const void* id, int rank, int nranks) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (ctx->dry()) fail(AMLT_ERR_NO_DEVICE, "amlt_gpu_comm_attach needs a device context");
        comm_release(ctx);
        // (a one-rank communicator is made too: its broadcasts are no-ops, but
        // the whole broadcast path runs, which is how one GPU tests it)
        if (!nccl().ok) fail(AMLT_ERR_CUDA, "libnccl.so.2 could not be loaded");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        NcclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        ncclComm_t c = nullptr;
        const int r = nccl().init_rank(&c, nranks, uid, rank);
        if (r != kNcclSuccess) fail(AMLT_ERR_CUDA, std::string("ncclCommInitRank: ") + nccl_error_string(r));
        comm_use(ctx, c, rank, nranks, true);
    });
}

amlt_status amlt_gpu_comm_detach(amlt_ctx* ctx) {
    if (!ctx) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] { comm_release(ctx); });
}

int amlt_gpu_comm_size(const amlt_ctx* ctx) { return ctx ? ctx->comm_size : 0; }

amlt_status amlt_gpu_last_host_layout(const amlt_ctx* ctx, int64_t* out) {
    if (!ctx || !out) return AMLT_ERR_INVALID_ARGUMENT;
    std::memcpy(out, ctx->host_layout, sizeof(ctx->host_layout));
    return AMLT_OK;
}

// ---------------------------------------------------------------------------
// device matrices for callers without their own allocator (SURVEY §8b
// "amlt_gpu_upload/alloc"): the reference's f64 MatrixBuffers in and out,
// stored on the device in the plan's dtype.

namespace {
void convert_rows(const double* src, void* dst, int64_t n, int dtype) {
    if (dtype == AMLT_F64) {
        std::memcpy(dst, src, size_t(n) * 8);
    } else if (dtype == AMLT_F32) {
        float* d = static_cast<float*>(dst);
        for (int64_t i = 0; i < n; ++i) d[i] = static_cast<float>(src[i]);
    } else {
        int32_t* d = static_cast<int32_t*>(dst);
        for (int64_t i = 0; i < n; ++i) d[i] = static_cast<int32_t>(src[i]);
    }
}
void widen_rows(const void* src, double* dst, int64_t n, int dtype) {
    if (dtype == AMLT_F64) {
        std::memcpy(dst, src, size_t(n) * 8);
    } else if (dtype == AMLT_F32) {
        const float* s = static_cast<const float*>(src);
        for (int64_t i = 0; i < n; ++i) dst[i] = s[i];
    } else {
        const int32_t* s = static_cast<const int32_t*>(src);
        for (int64_t i = 0; i < n; ++i) dst[i] = s[i];
    }
}
}  // namespace

amlt_status amlt_gpu_matrix_alloc(amlt_ctx* ctx, int64_t rows, int64_t cols, int order, int dtype,
                                  amlt_matrix* out) {
    if (!ctx || !out || rows < 0 || cols < 0 || (order != AMLT_ROW_MAJOR && order != AMLT_COL_MAJOR) ||
        dtype < AMLT_F64 || dtype > AMLT_I32)
        return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (ctx->dry()) fail(AMLT_ERR_NO_DEVICE, "amlt_gpu_matrix_alloc needs a device context");
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int es = dtype_size(dtype);
        const int64_t inner = order == AMLT_ROW_MAJOR ? cols : rows;
        const int64_t outer = order == AMLT_ROW_MAJOR ? rows : cols;
        // leading dimension padded to 16 bytes: TMA-staged (aligned) variants apply
        const int64_t vn = 16 / es;
        const int64_t ld = std::max<int64_t>((inner + vn - 1) / vn * vn, vn);
        void* p = nullptr;
        cuda_check(cudaMalloc(&p, size_t(std::max<int64_t>(outer, 1)) * size_t(ld) * es),
                   "cudaMalloc(matrix)");
        out->data = p;
        out->rows = rows;
        out->cols = cols;
        out->ld = ld;
        out->order = order;
        out->dtype = dtype;
    });
}

amlt_status amlt_gpu_matrix_free(amlt_ctx* ctx, amlt_matrix* m) {
    if (!ctx || !m) return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        if (m->data) {
            cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
            cuda_check(cudaFree(m->data), "cudaFree(matrix)");
        }
        m->data = nullptr;
    });
}

amlt_status amlt_gpu_matrix_upload(amlt_ctx* ctx, const amlt_matrix* dev, const double* host,
                                   int64_t host_ld) {
    if (!ctx || !dev || !dev->data || (!host && dev->rows * dev->cols > 0))
        return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int64_t inner = dev->order == AMLT_ROW_MAJOR ? dev->cols : dev->rows;
        const int64_t outer = dev->order == AMLT_ROW_MAJOR ? dev->rows : dev->cols;
        if (host_ld < inner) fail(AMLT_ERR_INVALID_ARGUMENT, "host leading dimension too small");
        if (inner == 0 || outer == 0) return;
        const int es = dtype_size(dev->dtype);
        std::vector<unsigned char> stage(size_t(outer) * size_t(dev->ld) * es, 0);
        for (int64_t o = 0; o < outer; ++o)
            convert_rows(host + o * host_ld, stage.data() + size_t(o) * size_t(dev->ld) * es, inner,
                         dev->dtype);
        cuda_check(cudaMemcpyAsync(dev->data, stage.data(), stage.size(), cudaMemcpyHostToDevice,
                                   ctx->stream),
                   "cudaMemcpyAsync H2D");
        cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
    });
}

amlt_status amlt_gpu_matrix_download(amlt_ctx* ctx, const amlt_matrix* dev, double* host,
                                     int64_t host_ld) {
    if (!ctx || !dev || !dev->data || (!host && dev->rows * dev->cols > 0))
        return AMLT_ERR_INVALID_ARGUMENT;
    return guarded(ctx, [&] {
        cuda_check(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int64_t inner = dev->order == AMLT_ROW_MAJOR ? dev->cols : dev->rows;
        const int64_t outer = dev->order == AMLT_ROW_MAJOR ? dev->rows : dev->cols;
        if (host_ld < inner) fail(AMLT_ERR_INVALID_ARGUMENT, "host leading dimension too small");
        if (inner == 0 || outer == 0) return;
        const int es = dtype_size(dev->dtype);
        std::vector<unsigned char> stage(size_t(outer) * size_t(dev->ld) * es);
        cuda_check(cudaMemcpyAsync(stage.data(), dev->data, stage.size(), cudaMemcpyDeviceToHost,
                                   ctx->stream),
                   "cudaMemcpyAsync D2H");
        cuda_check(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
        for (int64_t o = 0; o < outer; ++o)
            widen_rows(stage.data() + size_t(o) * size_t(dev->ld) * es, host + o * host_ld, inner,
                       dev->dtype);
    });
}

amlt_status amlt_spr(int64_t M, int64_t K, int64_t N, double seconds, double* out) {
    if (!out) return AMLT_ERR_INVALID_ARGUMENT;
    if (!(seconds > 0.0)) return AMLT_ERR_NON_POSITIVE_TIME;
    *out = double(M) * double(K) * double(N) / (1e9 * seconds);
    return AMLT_OK;
}

}  // extern "C"
