// sharded.cu — single-process row-band multi-GPU execution (amlt_gpu_run_sharded).
//
// The GPU counterpart of running the reference's adaptive_execute on row
// bands (its own all-cores mode): device d owns rows
// [M d/n, M (d+1)/n) of A and R; B and the per-column vectors are replicated
// with NCCL broadcasts from devices[0] over NVLink 5 / NVSwitch; no
// reduction. NCCL is loaded with dlopen so the library has no link-time NCCL
// dependency (and shares torch's NCCL when torch already loaded one).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/amlt_gpu.h"

namespace {

// --- minimal NCCL surface (nccl.h), resolved at run time
using ncclComm_t = struct ncclComm*;
enum { ncclSuccess = 0 };
enum { ncclInt8 = 0, ncclUint8 = 1, ncclInt32 = 2, ncclFloat32 = 7, ncclFloat64 = 8 };
using PInitAll = int (*)(ncclComm_t*, int, const int*);
using PBcast = int (*)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t);
using PGroup = int (*)();
using PDestroy = int (*)(ncclComm_t);
using PErr = const char* (*)(int);

struct Nccl {
    PInitAll init_all = nullptr;
    PBcast bcast = nullptr;
    PGroup group_start = nullptr, group_end = nullptr;
    PDestroy destroy = nullptr;
    PErr err = nullptr;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        n.init_all = reinterpret_cast<PInitAll>(dlsym(h, "ncclCommInitAll"));
        n.bcast = reinterpret_cast<PBcast>(dlsym(h, "ncclBroadcast"));
        n.group_start = reinterpret_cast<PGroup>(dlsym(h, "ncclGroupStart"));
        n.group_end = reinterpret_cast<PGroup>(dlsym(h, "ncclGroupEnd"));
        n.destroy = reinterpret_cast<PDestroy>(dlsym(h, "ncclCommDestroy"));
        n.err = reinterpret_cast<PErr>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.init_all && n.bcast && n.group_start && n.group_end && n.destroy;
    });
    return n;
}

struct Fail : std::runtime_error {
    amlt_status code;
    Fail(amlt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Fail(AMLT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void nk(int r, const char* what) {
    if (r != ncclSuccess)
        throw Fail(AMLT_ERR_CUDA, std::string(what) + ": " + (nccl().err ? nccl().err(r) : "NCCL error"));
}

int es_of(int dt) { return dt == AMLT_F64 ? 8 : 4; }
size_t bytes_of(const amlt_matrix& m) {
    if (!m.data) return 0;
    const int64_t outer = m.order == AMLT_ROW_MAJOR ? m.rows : m.cols;
    return size_t(std::max<int64_t>(outer, 1)) * size_t(m.ld) * es_of(m.dtype);
}

struct DevState {
    int device = 0;
    amlt_ctx* ctx = nullptr;
    amlt_plan* plan = nullptr;
    cudaStream_t stream = nullptr;
    void* buf[3] = {nullptr, nullptr, nullptr};  // A band, B, R band
    std::vector<void*> xbuf;                     // per extra operand (see Extra)
    int64_t r0 = 0, r1 = 0;
    amlt_status st = AMLT_OK;
    std::string err;
};

// An operand besides A / B / R: thres, dis or a generated body's aux leaf.
// Leaves indexed by i follow the row split: a row-major [i][j] matrix is
// copied band by band like R; an [i] vector (or a col-major [i][j]) is
// replicated and viewed from row r0. Everything else is replicated.
struct Extra {
    const amlt_matrix* host = nullptr;
    int cls = AMLT_LEAF_VEC_J;
    bool banded = false;  // row-major [i][j]: per-device band copies
    size_t bytes = 0;     // replicated copy size
};

int64_t vec_step(const amlt_matrix& t) {
    return (t.cols == 1) ? (t.order == AMLT_ROW_MAJOR ? t.ld : 1) : (t.order == AMLT_ROW_MAJOR ? 1 : t.ld);
}

// The device view of an extra operand on the device owning rows [r0, r1).
amlt_matrix band_view(const Extra& x, void* dev, int64_t r0, int64_t r1) {
    amlt_matrix m = *x.host;
    m.data = dev;
    if (!dev) return m;
    const int es = es_of(m.dtype);
    if (x.cls == AMLT_LEAF_VEC_I) {
        m.data = static_cast<char*>(dev) + r0 * vec_step(*x.host) * es;
        if (m.cols == 1) m.rows = std::max<int64_t>(m.rows - r0, 0);
        else m.cols = std::max<int64_t>(m.cols - r0, 0);
    } else if (x.cls == AMLT_LEAF_MAT_IJ) {
        if (x.banded) {
            m.rows = r1 - r0;
        } else {  // col-major: element (i, j) at i + j * ld
            m.data = static_cast<char*>(dev) + r0 * es;
            m.rows = std::max<int64_t>(m.rows - r0, 0);
        }
    }
    return m;
}

thread_local std::string g_sharded_error;

// Shared by the body-descriptor and task-text entries: make_plan creates
// the per-device plan (and reports the aux classes of generated bodies).
template <class MakePlan>
amlt_status run_sharded_impl(int dtype, int layout_a, int thres_class, MakePlan make_plan,
                             const amlt_operands* ho, const amlt_bounds* bounds, int n,
                             const int* devices, int flags, double* elapsed_s) {
    std::vector<DevState> ds(static_cast<size_t>(n));
    std::vector<ncclComm_t> comms;
    auto cleanup = [&] {
        for (auto& d : ds) {
            if (d.device >= 0) cudaSetDevice(d.device);
            if (d.stream) cudaStreamSynchronize(d.stream);
            for (void* p : d.buf)
                if (p) cudaFree(p);
            for (void* p : d.xbuf)
                if (p) cudaFree(p);
            if (d.plan) amlt_gpu_plan_destroy(d.plan);
            if (d.ctx) amlt_gpu_ctx_destroy(d.ctx);
            if (d.stream) cudaStreamDestroy(d.stream);
        }
        for (auto c : comms)
            if (c) nccl().destroy(c);
    };
    try {
        const int es = es_of(dtype);
        const int64_t M = bounds->i1 - bounds->i0;
        // A: each statement row i must be a contiguous run along k (row stride lda)
        const bool a_rows = (layout_a == AMLT_LAYOUT_NORMAL && ho->a.order == AMLT_ROW_MAJOR) ||
                            (layout_a == AMLT_LAYOUT_TRANSPOSED && ho->a.order == AMLT_COL_MAJOR);
        if (!a_rows || ho->r.order != AMLT_ROW_MAJOR)
            throw Fail(AMLT_ERR_UNSUPPORTED,
                       "run_sharded needs A rows (k) contiguous and a row-major R; use run_host per device");
        if (M < 0) throw Fail(AMLT_ERR_INVALID_ARGUMENT, "bad bounds");
        if (n > 1 && !nccl().ok) throw Fail(AMLT_ERR_CUDA, "libnccl.so.2 could not be loaded");

        const size_t bB = bytes_of(ho->b);
        const int64_t a_ld = ho->a.ld, r_ld = ho->r.ld;
        std::vector<int> aux_class;
        for (int d = 0; d < n; ++d) {
            DevState& s = ds[static_cast<size_t>(d)];
            s.device = devices[d];
            s.r0 = bounds->i0 + M * d / n;
            s.r1 = bounds->i0 + M * (d + 1) / n;
            amlt_status st = amlt_gpu_ctx_create(s.device, 0, &s.ctx);
            if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(nullptr));
            st = make_plan(s.ctx, &s.plan, &aux_class);
            if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(s.ctx));
        }
        // the extra operands: thres, dis, then the aux leaves by position
        std::vector<Extra> ex;
        auto add_extra = [&](const amlt_matrix* m, int cls) {
            Extra x;
            x.host = m;
            x.cls = cls;
            x.banded = cls == AMLT_LEAF_MAT_IJ && m->order == AMLT_ROW_MAJOR;
            x.bytes = x.banded ? 0 : bytes_of(*m);
            ex.push_back(x);
        };
        add_extra(&ho->thres, thres_class);
        add_extra(&ho->dis, AMLT_LEAF_VEC_J);
        for (size_t q = 0; q < aux_class.size() && static_cast<int>(q) < ho->n_aux; ++q)
            add_extra(&ho->aux[q], aux_class[q]);
        for (auto& s : ds) {
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
            amlt_gpu_set_stream(s.ctx, s.stream);
            const size_t rows = size_t(s.r1 - s.r0);
            // the A band keeps the buffer's own row pitch; rows [r0, r1) only
            ck(cudaMalloc(&s.buf[0], std::max<size_t>(rows, 1) * a_ld * es), "cudaMalloc A band");
            ck(cudaMalloc(&s.buf[1], std::max<size_t>(bB, 16)), "cudaMalloc B");
            ck(cudaMalloc(&s.buf[2], std::max<size_t>(rows, 1) * r_ld * es), "cudaMalloc R band");
            s.xbuf.assign(ex.size(), nullptr);
            for (size_t x = 0; x < ex.size(); ++x) {
                if (!ex[x].host->data) continue;
                const size_t b = ex[x].banded ? std::max<size_t>(rows, 1) * ex[x].host->ld * es : ex[x].bytes;
                ck(cudaMalloc(&s.xbuf[x], std::max<size_t>(b, 16)), "cudaMalloc extra operand");
            }
        }
        if (n > 1) {
            comms.assign(static_cast<size_t>(n), nullptr);
            nk(nccl().init_all(comms.data(), n, devices), "ncclCommInitAll");
        }

        auto t0 = std::chrono::steady_clock::now();
        // H2D: A / R (and row-major [i][j]) bands to their owners, B and the
        // replicated operands to devices[0]
        for (int d = 0; d < n; ++d) {
            DevState& s = ds[static_cast<size_t>(d)];
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            const size_t rows = size_t(s.r1 - s.r0);
            const char* a_src = static_cast<const char*>(ho->a.data) + size_t(s.r0) * a_ld * es;
            ck(cudaMemcpyAsync(s.buf[0], a_src, rows * a_ld * es, cudaMemcpyHostToDevice, s.stream),
               "H2D A band");
            char* r_src = static_cast<char*>(ho->r.data) + size_t(s.r0) * r_ld * es;
            if (flags & AMLT_HOST_R_ZERO)
                ck(cudaMemsetAsync(s.buf[2], 0, rows * r_ld * es, s.stream), "memset R band");
            else
                ck(cudaMemcpyAsync(s.buf[2], r_src, rows * r_ld * es, cudaMemcpyHostToDevice, s.stream),
                   "H2D R band");
            for (size_t x = 0; x < ex.size(); ++x) {
                const amlt_matrix& m = *ex[x].host;
                if (!m.data) continue;
                if (ex[x].banded) {
                    const size_t pitch = size_t(m.ld) * es;
                    ck(cudaMemcpyAsync(s.xbuf[x], static_cast<const char*>(m.data) + size_t(s.r0) * pitch,
                                       rows * pitch, cudaMemcpyHostToDevice, s.stream),
                       "H2D [i][j] band");
                } else if (d == 0) {
                    ck(cudaMemcpyAsync(s.xbuf[x], m.data, ex[x].bytes, cudaMemcpyHostToDevice, s.stream),
                       "H2D replicated operand");
                }
            }
            if (d == 0)
                ck(cudaMemcpyAsync(s.buf[1], ho->b.data, bB, cudaMemcpyHostToDevice, s.stream), "H2D B");
        }
        // replicate B and the replicated operands over NVLink (one group)
        if (n > 1) {
            nk(nccl().group_start(), "ncclGroupStart");
            for (int d = 0; d < n; ++d) {
                DevState& s = ds[static_cast<size_t>(d)];
                nk(nccl().bcast(s.buf[1], s.buf[1], bB, ncclUint8, 0, comms[static_cast<size_t>(d)],
                                s.stream),
                   "ncclBroadcast");
                for (size_t x = 0; x < ex.size(); ++x) {
                    if (!ex[x].host->data || ex[x].banded || !ex[x].bytes) continue;
                    nk(nccl().bcast(s.xbuf[x], s.xbuf[x], ex[x].bytes, ncclUint8, 0,
                                    comms[static_cast<size_t>(d)], s.stream),
                       "ncclBroadcast");
                }
            }
            nk(nccl().group_end(), "ncclGroupEnd");
        }
        // compute: one host thread per device, each its own band
        std::vector<std::thread> th;
        for (int d = 0; d < n; ++d) {
            th.emplace_back([&, d] {
                DevState& s = ds[static_cast<size_t>(d)];
                cudaSetDevice(s.device);
                amlt_operands o = *ho;
                o.a.data = s.buf[0];
                o.a.rows = ho->a.order == AMLT_ROW_MAJOR ? (s.r1 - s.r0) : ho->a.rows;
                o.a.cols = ho->a.order == AMLT_ROW_MAJOR ? ho->a.cols : (s.r1 - s.r0);
                o.b.data = s.buf[1];
                o.r.data = s.buf[2];
                o.r.rows = s.r1 - s.r0;
                o.thres = band_view(ex[0], s.xbuf[0], s.r0, s.r1);
                o.dis = band_view(ex[1], s.xbuf[1], s.r0, s.r1);
                for (size_t q = 2; q < ex.size(); ++q)
                    o.aux[q - 2] = band_view(ex[q], s.xbuf[q], s.r0, s.r1);
                // band-local bounds: rows [0, r1 - r0), same j / k ranges
                amlt_bounds bb = *bounds;
                bb.i0 = 0;
                bb.i1 = s.r1 - s.r0;
                if (bb.i1 > 0) {
                    amlt_tune_report rep;
                    s.st = amlt_gpu_adaptive_execute(s.ctx, s.plan, &o, &bb, 0, nullptr, nullptr,
                                                     nullptr, &rep);
                    if (s.st != AMLT_OK) s.err = amlt_gpu_last_error(s.ctx);
                }
            });
        }
        for (auto& t : th) t.join();
        for (auto& s : ds)
            if (s.st != AMLT_OK) throw Fail(s.st, s.err);
        // D2H R bands
        for (auto& s : ds) {
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            const size_t rows = size_t(s.r1 - s.r0);
            char* r_dst = static_cast<char*>(ho->r.data) + size_t(s.r0) * r_ld * es;
            ck(cudaMemcpyAsync(r_dst, s.buf[2], rows * r_ld * es, cudaMemcpyDeviceToHost, s.stream),
               "D2H R band");
        }
        for (auto& s : ds) {
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            ck(cudaStreamSynchronize(s.stream), "cudaStreamSynchronize");
        }
        auto t1 = std::chrono::steady_clock::now();
        if (elapsed_s) *elapsed_s = std::chrono::duration<double>(t1 - t0).count();
        cleanup();
        g_sharded_error.clear();
        return AMLT_OK;
    } catch (const Fail& e) {
        g_sharded_error = e.what();
        cleanup();
        return e.code;
    } catch (const std::exception& e) {
        g_sharded_error = e.what();
        cleanup();
        return AMLT_ERR_ENGINE;
    }
}

}  // namespace

extern "C" amlt_status amlt_gpu_run_sharded(const amlt_body_desc* desc, const amlt_operands* ho,
                                            const amlt_bounds* bounds, int n, const int* devices,
                                            int flags, double* elapsed_s) {
    if (!desc || !ho || !bounds || n < 1 || !devices) return AMLT_ERR_INVALID_ARGUMENT;
    const bool needs_t = desc->body == AMLT_BODY_DISCOUNT || desc->body == AMLT_BODY_BOOST ||
                         desc->body == AMLT_BODY_THRCOUNT;
    return run_sharded_impl(
        desc->dtype, desc->layout_a, needs_t ? desc->thres_class : AMLT_LEAF_VEC_J,
        [&](amlt_ctx* ctx, amlt_plan** plan, std::vector<int>*) {
            return amlt_gpu_plan_create(ctx, desc, plan);
        },
        ho, bounds, n, devices, flags, elapsed_s);
}

extern "C" amlt_status amlt_gpu_run_sharded_source(const char* task_source, int dtype,
                                                   const amlt_operands* ho, const amlt_bounds* bounds,
                                                   int n, const int* devices, int flags,
                                                   double* elapsed_s) {
    if (!task_source || !ho || !bounds || n < 1 || !devices) return AMLT_ERR_INVALID_ARGUMENT;
    amlt_task_info info;
    amlt_status st = amlt_gpu_recognize(task_source, &info);
    if (st != AMLT_OK) {
        g_sharded_error = amlt_gpu_last_error(nullptr);
        return st;
    }
    const bool needs_t = info.desc.body == AMLT_BODY_DISCOUNT || info.desc.body == AMLT_BODY_BOOST ||
                         info.desc.body == AMLT_BODY_THRCOUNT;
    return run_sharded_impl(
        dtype, info.desc.layout_a, needs_t ? info.desc.thres_class : AMLT_LEAF_VEC_J,
        [&](amlt_ctx* ctx, amlt_plan** plan, std::vector<int>* aux_class) {
            amlt_task_info ti;
            amlt_status r = amlt_gpu_plan_from_source(ctx, task_source, dtype, plan, &ti);
            if (r == AMLT_OK) aux_class->assign(ti.aux_class, ti.aux_class + ti.n_aux);
            return r;
        },
        ho, bounds, n, devices, flags, elapsed_s);
}

extern "C" const char* amlt_gpu_sharded_last_error(void) { return g_sharded_error.c_str(); }
