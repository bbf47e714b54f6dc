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
    void* buf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};  // A band, B, R band, thres, dis
    int64_t r0 = 0, r1 = 0;
    amlt_status st = AMLT_OK;
    std::string err;
};

}  // namespace

thread_local std::string g_sharded_error;

extern "C" amlt_status amlt_gpu_run_sharded(const amlt_body_desc* desc, const amlt_operands* ho,
                                            const amlt_bounds* bounds, int n, const int* devices,
                                            int flags, double* elapsed_s) {
    if (!desc || !ho || !bounds || n < 1 || !devices) return AMLT_ERR_INVALID_ARGUMENT;
    std::vector<DevState> ds(static_cast<size_t>(n));
    std::vector<ncclComm_t> comms;
    auto cleanup = [&] {
        for (auto& d : ds) {
            if (d.device >= 0) cudaSetDevice(d.device);
            if (d.stream) cudaStreamSynchronize(d.stream);
            for (void* p : d.buf)
                if (p) cudaFree(p);
            if (d.plan) amlt_gpu_plan_destroy(d.plan);
            if (d.ctx) amlt_gpu_ctx_destroy(d.ctx);
            if (d.stream) cudaStreamDestroy(d.stream);
        }
        for (auto c : comms)
            if (c) nccl().destroy(c);
    };
    try {
        const amlt_body_desc& bd = *desc;
        const int es = es_of(bd.dtype);
        const int64_t M = bounds->i1 - bounds->i0;
        // A: each statement row i must be a contiguous run along k (row stride lda)
        const bool a_rows = (bd.layout_a == AMLT_LAYOUT_NORMAL && ho->a.order == AMLT_ROW_MAJOR) ||
                            (bd.layout_a == AMLT_LAYOUT_TRANSPOSED && ho->a.order == AMLT_COL_MAJOR);
        if (!a_rows || ho->r.order != AMLT_ROW_MAJOR)
            throw Fail(AMLT_ERR_UNSUPPORTED,
                       "run_sharded needs A rows (k) contiguous and a row-major R; use run_host per device");
        if (M < 0) throw Fail(AMLT_ERR_INVALID_ARGUMENT, "bad bounds");
        if (n > 1 && !nccl().ok) throw Fail(AMLT_ERR_CUDA, "libnccl.so.2 could not be loaded");

        const size_t bB = bytes_of(ho->b), bT = bytes_of(ho->thres), bD = bytes_of(ho->dis);
        const int64_t a_ld = ho->a.ld, r_ld = ho->r.ld;
        for (int d = 0; d < n; ++d) {
            DevState& s = ds[static_cast<size_t>(d)];
            s.device = devices[d];
            s.r0 = bounds->i0 + M * d / n;
            s.r1 = bounds->i0 + M * (d + 1) / n;
            amlt_status st = amlt_gpu_ctx_create(s.device, 0, &s.ctx);
            if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(nullptr));
            st = amlt_gpu_plan_create(s.ctx, &bd, &s.plan);
            if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(s.ctx));
            ck(cudaSetDevice(s.device), "cudaSetDevice");
            ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "cudaStreamCreate");
            amlt_gpu_set_stream(s.ctx, s.stream);
            const size_t rows = size_t(s.r1 - s.r0);
            // the A band keeps the buffer's own row pitch; rows [r0, r1) only
            ck(cudaMalloc(&s.buf[0], std::max<size_t>(rows, 1) * a_ld * es), "cudaMalloc A band");
            ck(cudaMalloc(&s.buf[1], std::max<size_t>(bB, 16)), "cudaMalloc B");
            ck(cudaMalloc(&s.buf[2], std::max<size_t>(rows, 1) * r_ld * es), "cudaMalloc R band");
            if (bT) ck(cudaMalloc(&s.buf[3], bT), "cudaMalloc thres");
            if (bD) ck(cudaMalloc(&s.buf[4], bD), "cudaMalloc dis");
        }
        if (n > 1) {
            comms.assign(static_cast<size_t>(n), nullptr);
            nk(nccl().init_all(comms.data(), n, devices), "ncclCommInitAll");
        }

        auto t0 = std::chrono::steady_clock::now();
        // H2D: A / R bands to their owners, B and the vectors to devices[0]
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
            if (d == 0) {
                ck(cudaMemcpyAsync(s.buf[1], ho->b.data, bB, cudaMemcpyHostToDevice, s.stream), "H2D B");
                if (bT)
                    ck(cudaMemcpyAsync(s.buf[3], ho->thres.data, bT, cudaMemcpyHostToDevice, s.stream),
                       "H2D thres");
                if (bD)
                    ck(cudaMemcpyAsync(s.buf[4], ho->dis.data, bD, cudaMemcpyHostToDevice, s.stream),
                       "H2D dis");
            }
        }
        // replicate B / thres / dis over NVLink (byte broadcasts, in one group)
        if (n > 1) {
            nk(nccl().group_start(), "ncclGroupStart");
            for (int slot : {1, 3, 4}) {
                const size_t bytes = slot == 1 ? bB : slot == 3 ? bT : bD;
                if (!bytes) continue;
                for (int d = 0; d < n; ++d) {
                    DevState& s = ds[static_cast<size_t>(d)];
                    nk(nccl().bcast(s.buf[slot], s.buf[slot], bytes, ncclUint8, 0,
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
                o.thres.data = s.buf[3];
                o.dis.data = s.buf[4];
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

extern "C" const char* amlt_gpu_sharded_last_error(void) { return g_sharded_error.c_str(); }
