// sharded.cu — single-process row-band multi-GPU execution: the persistent
// group (amlt_sharded_*) and the one-shot amlt_gpu_run_sharded(_source).
//
// The GPU counterpart of running the reference's adaptive_execute on row
// bands (its own all-cores mode): device d owns rows
// [M d/n, M (d+1)/n) of A and R (edges on 64-row multiples); B and the
// per-column vectors are read from host memory by device 0 only and
// broadcast (NCCL over NVLink 5 / NVSwitch) panel by panel inside each
// device's host pipeline (amlt_gpu_run_host_adaptive with
// AMLT_HOST_BCAST_SHARED), so the transfers overlap compute; no reduction.
// The group keeps its contexts, communicator, plans and tuning winners
// across runs: only the first run of a shape tunes.
#include <cuda_runtime.h>

#include <chrono>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/amlt_gpu.h"
#include "nccl_dl.h"

namespace amltk {
amlt_status ctx_use_comm(amlt_ctx* ctx, void* comm, int rank, int nranks);
}

using namespace amltk;

struct amlt_sharded {
    bool dry = false;  // AMLT_CTX_DRY_RUN: contexts without devices; runs validate and plan only
    std::vector<int> devices;
    std::vector<amlt_ctx*> ctx;
    std::vector<ncclComm_t> comms;
    // plans per device, by body description or task text
    std::map<std::string, std::vector<amlt_plan*>> plans;
    std::vector<std::vector<int>> aux_class;  // per plan key (generated bodies)
    std::map<std::string, size_t> aux_index;
    std::string err;
    std::mutex mu;
};

namespace {

struct Fail : std::runtime_error {
    amlt_status code;
    Fail(amlt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

thread_local std::string g_sharded_error;
thread_local std::string g_group_create_error;

int64_t vec_step(const amlt_matrix& t) {
    return (t.cols == 1) ? (t.order == AMLT_ROW_MAJOR ? t.ld : 1) : (t.order == AMLT_ROW_MAJOR ? 1 : t.ld);
}

// The band view of an operand indexed by i (an [i] vector or an [i][j]
// matrix) for rows [r0, r1): the same host buffer, offset to row r0.
amlt_matrix band_view(const amlt_matrix& h, int cls, int64_t r0, int64_t r1) {
    amlt_matrix m = h;
    if (!h.data) return m;
    const int es = h.dtype == AMLT_F64 ? 8 : 4;
    if (cls == AMLT_LEAF_VEC_I) {
        m.data = static_cast<char*>(h.data) + r0 * vec_step(h) * es;
        if (m.cols == 1) m.rows = std::max<int64_t>(r1 - r0, 0);
        else m.cols = std::max<int64_t>(r1 - r0, 0);
    } else if (cls == AMLT_LEAF_MAT_IJ) {
        if (h.order == AMLT_ROW_MAJOR) {
            m.data = static_cast<char*>(h.data) + r0 * h.ld * es;
        } else {
            m.data = static_cast<char*>(h.data) + r0 * es;
        }
        m.rows = std::max<int64_t>(r1 - r0, 0);
    }
    return m;
}

std::string desc_key(const amlt_body_desc& d) {
    return "desc:" + std::string(reinterpret_cast<const char*>(&d), sizeof(d));
}

// Plans for every device of the group (made on first use).
const std::vector<amlt_plan*>& group_plans(amlt_sharded* g, const amlt_body_desc* desc, const char* src,
                                           int dtype, std::vector<int>* aux_class, amlt_task_info* info) {
    amlt_body_desc dd{};
    if (!src) {
        dd = *desc;
        dd.dtype = dtype;
    }
    const std::string key = src ? "src:" + std::to_string(dtype) + ":" + src : desc_key(dd);
    amlt_task_info ti{};
    if (src) {
        const amlt_status st = amlt_gpu_recognize(src, &ti);
        if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(nullptr));
    } else {
        ti.desc = dd;
    }
    if (info) *info = ti;
    auto it = g->plans.find(key);
    if (it == g->plans.end()) {
        std::vector<amlt_plan*> ps(g->ctx.size(), nullptr);
        std::vector<int> ac;
        for (size_t d = 0; d < g->ctx.size(); ++d) {
            amlt_status st;
            if (src) {
                amlt_task_info t2;
                st = amlt_gpu_plan_from_source(g->ctx[d], src, dtype, &ps[d], &t2);
                if (st == AMLT_OK) ac.assign(t2.aux_class, t2.aux_class + t2.n_aux);
            } else {
                st = amlt_gpu_plan_create(g->ctx[d], &dd, &ps[d]);
            }
            if (st != AMLT_OK) {
                std::string m = amlt_gpu_last_error(g->ctx[d]);
                for (auto* p : ps)
                    if (p) amlt_gpu_plan_destroy(p);
                throw Fail(st, m);
            }
        }
        it = g->plans.emplace(key, std::move(ps)).first;
        g->aux_index[key] = g->aux_class.size();
        g->aux_class.push_back(ac);
    }
    if (aux_class) *aux_class = g->aux_class[g->aux_index[key]];
    return it->second;
}

amlt_status group_run(amlt_sharded* g, const amlt_body_desc* desc, const char* src, int dtype,
                      const amlt_operands* ho, const amlt_bounds* bounds, int flags, amlt_tune_report* reports,
                      double* elapsed_s) {
    std::lock_guard<std::mutex> lock(g->mu);  // one run at a time per group
    try {
        std::vector<int> aux_class;
        amlt_task_info info{};
        const std::vector<amlt_plan*>& plans = group_plans(g, desc, src, dtype, &aux_class, &info);
        const amlt_body_desc& bd = info.desc;
        const int n = static_cast<int>(g->ctx.size());
        const int64_t M = bounds->i1 - bounds->i0;
        if (M < 0) throw Fail(AMLT_ERR_INVALID_ARGUMENT, "bad bounds");
        // A: each statement row i a contiguous run along k; R row-major
        const bool a_rows = (bd.layout_a == AMLT_LAYOUT_NORMAL && ho->a.order == AMLT_ROW_MAJOR) ||
                            (bd.layout_a == AMLT_LAYOUT_TRANSPOSED && ho->a.order == AMLT_COL_MAJOR);
        if (!a_rows || ho->r.order != AMLT_ROW_MAJOR)
            throw Fail(AMLT_ERR_UNSUPPORTED,
                       "sharded runs need A rows (k) contiguous and a row-major R; use run_host per device");
        const int es = ho->a.dtype == AMLT_F64 ? 8 : 4;
        const bool needs_t = bd.body == AMLT_BODY_DISCOUNT || bd.body == AMLT_BODY_BOOST ||
                             bd.body == AMLT_BODY_THRCOUNT;
        const int tcls = needs_t ? bd.thres_class : AMLT_LEAF_VEC_J;
        // band edges on 64-row multiples (tile-aligned for every variant height)
        std::vector<int64_t> edge(static_cast<size_t>(n) + 1);
        for (int d = 0; d <= n; ++d) {
            int64_t e = d == n ? M : (M * d / n + 32) / 64 * 64;
            edge[static_cast<size_t>(d)] = bounds->i0 + std::min<int64_t>(M, std::max<int64_t>(0, e));
        }
        std::vector<amlt_status> st(static_cast<size_t>(n), AMLT_OK);
        std::vector<std::string> msg(static_cast<size_t>(n));
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int d = 0; d < n; ++d) {
            th.emplace_back([&, d] {
                const int64_t r0 = edge[static_cast<size_t>(d)], r1 = edge[static_cast<size_t>(d) + 1];
                amlt_operands o = *ho;
                // this device's rows of A and R: the host buffers offset to row r0
                if (ho->a.order == AMLT_ROW_MAJOR) {
                    o.a.data = static_cast<char*>(ho->a.data) + r0 * ho->a.ld * es;
                    o.a.rows = r1 - r0;
                } else {
                    o.a.data = static_cast<char*>(ho->a.data) + r0 * ho->a.ld * es;
                    o.a.cols = r1 - r0;
                }
                o.r.data = static_cast<char*>(ho->r.data) + r0 * ho->r.ld * es;
                o.r.rows = r1 - r0;
                o.thres = band_view(ho->thres, tcls, r0, r1);
                for (size_t q = 0; q < aux_class.size() && static_cast<int>(q) < ho->n_aux; ++q)
                    o.aux[q] = band_view(ho->aux[q], aux_class[q], r0, r1);
                amlt_bounds bb = *bounds;
                bb.i0 = 0;
                bb.i1 = r1 - r0;
                amlt_tune_report local;
                amlt_tune_report* rep = reports ? &reports[d] : &local;
                std::memset(rep, 0, sizeof(*rep));
                if (g->dry) {
                    // plan and validate the band's operands (no device): one
                    // subtask over the band, its rectangle reported
                    st[static_cast<size_t>(d)] = amlt_gpu_run_subtask(
                        g->ctx[static_cast<size_t>(d)], plans[static_cast<size_t>(d)], &o, nullptr, &bb, nullptr,
                        nullptr, nullptr, nullptr);
                    rep->n_cover = 1;
                    rep->coverage[0] = amlt_cover_rect{r0, r1, bb.k0, bb.k1, bb.j0, bb.j1};
                } else {
                    // every rank takes part in the broadcasts, an empty band too
                    st[static_cast<size_t>(d)] = amlt_gpu_run_host_adaptive(
                        g->ctx[static_cast<size_t>(d)], plans[static_cast<size_t>(d)], &o, &bb,
                        flags | (n > 1 ? AMLT_HOST_BCAST_SHARED : 0), nullptr, nullptr, rep, nullptr);
                }
                if (st[static_cast<size_t>(d)] != AMLT_OK)
                    msg[static_cast<size_t>(d)] = amlt_gpu_last_error(g->ctx[static_cast<size_t>(d)]);
            });
        }
        for (auto& t : th) t.join();
        for (int d = 0; d < n; ++d)
            if (st[static_cast<size_t>(d)] != AMLT_OK)
                throw Fail(st[static_cast<size_t>(d)], "device " + std::to_string(g->devices[static_cast<size_t>(d)]) +
                                                           ": " + msg[static_cast<size_t>(d)]);
        auto t1 = std::chrono::steady_clock::now();
        if (elapsed_s) *elapsed_s = std::chrono::duration<double>(t1 - t0).count();
        g->err.clear();
        return AMLT_OK;
    } catch (const Fail& e) {
        g->err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g->err = e.what();
        return AMLT_ERR_ENGINE;
    }
}

}  // namespace

extern "C" {

amlt_status amlt_sharded_create(int n, const int* devices, int ctx_flags, amlt_sharded** out) {
    if (n < 1 || !devices || !out) return AMLT_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    auto g = std::make_unique<amlt_sharded>();
    try {
        g->dry = (ctx_flags & AMLT_CTX_DRY_RUN) != 0;
        g->devices.assign(devices, devices + n);
        for (int d = 0; d < n; ++d) {
            amlt_ctx* c = nullptr;
            const amlt_status st = amlt_gpu_ctx_create(devices[d], ctx_flags, &c);
            if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(nullptr));
            g->ctx.push_back(c);
        }
        if (n > 1 && !g->dry) {
            if (!nccl().ok) throw Fail(AMLT_ERR_CUDA, "libnccl.so.2 could not be loaded");
            g->comms.assign(static_cast<size_t>(n), nullptr);
            const int r = nccl().init_all(g->comms.data(), n, devices);
            if (r != kNcclSuccess) throw Fail(AMLT_ERR_CUDA, std::string("ncclCommInitAll: ") + nccl_error_string(r));
            for (int d = 0; d < n; ++d) {
                const amlt_status st = ctx_use_comm(g->ctx[static_cast<size_t>(d)], g->comms[static_cast<size_t>(d)], d, n);
                if (st != AMLT_OK) throw Fail(st, amlt_gpu_last_error(g->ctx[static_cast<size_t>(d)]));
            }
        }
    } catch (const Fail& e) {
        g_group_create_error = e.what();
        amlt_sharded_destroy(g.release());
        return e.code;
    }
    g_group_create_error.clear();
    *out = g.release();
    return AMLT_OK;
}

void amlt_sharded_destroy(amlt_sharded* g) {
    if (!g) return;
    for (auto& kv : g->plans)
        for (amlt_plan* p : kv.second)
            if (p) amlt_gpu_plan_destroy(p);
    for (size_t d = 0; d < g->ctx.size(); ++d) {
        if (d < g->comms.size() && g->comms[d]) amlt_gpu_comm_detach(g->ctx[d]);  // (not owned by the context)
        amlt_gpu_ctx_destroy(g->ctx[d]);
    }
    for (size_t d = 0; d < g->comms.size(); ++d)
        if (g->comms[d]) {
            cudaSetDevice(g->devices[d]);
            nccl().destroy(g->comms[d]);
        }
    delete g;
}

amlt_status amlt_sharded_run(amlt_sharded* g, const amlt_body_desc* desc, const char* task_source, int dtype,
                             const amlt_operands* host_ops, const amlt_bounds* bounds, int flags,
                             amlt_tune_report* reports, double* elapsed_s) {
    if (!g || (!desc && !task_source) || !host_ops || !bounds) return AMLT_ERR_INVALID_ARGUMENT;
    return group_run(g, desc, task_source, dtype, host_ops, bounds, flags, reports, elapsed_s);
}

int amlt_sharded_size(const amlt_sharded* g) { return g ? static_cast<int>(g->ctx.size()) : 0; }

const char* amlt_sharded_last_error(const amlt_sharded* g) {
    return g ? g->err.c_str() : g_group_create_error.c_str();
}

// One-shot forms: a group made for the call and destroyed after it.
amlt_status amlt_gpu_run_sharded(const amlt_body_desc* desc, const amlt_operands* ho, const amlt_bounds* bounds,
                                 int n, const int* devices, int flags, double* elapsed_s) {
    if (!desc || !ho || !bounds || n < 1 || !devices) return AMLT_ERR_INVALID_ARGUMENT;
    amlt_sharded* g = nullptr;
    amlt_status st = amlt_sharded_create(n, devices, 0, &g);
    if (st != AMLT_OK) {
        g_sharded_error = amlt_sharded_last_error(nullptr);
        return st;
    }
    st = amlt_sharded_run(g, desc, nullptr, desc->dtype, ho, bounds, flags, nullptr, elapsed_s);
    g_sharded_error = st == AMLT_OK ? "" : g->err;
    amlt_sharded_destroy(g);
    return st;
}

amlt_status amlt_gpu_run_sharded_source(const char* task_source, int dtype, const amlt_operands* ho,
                                        const amlt_bounds* bounds, int n, const int* devices, int flags,
                                        double* elapsed_s) {
    if (!task_source || !ho || !bounds || n < 1 || !devices) return AMLT_ERR_INVALID_ARGUMENT;
    amlt_task_info info;
    amlt_status st = amlt_gpu_recognize(task_source, &info);
    if (st != AMLT_OK) {
        g_sharded_error = amlt_gpu_last_error(nullptr);
        return st;
    }
    amlt_sharded* g = nullptr;
    st = amlt_sharded_create(n, devices, 0, &g);
    if (st != AMLT_OK) {
        g_sharded_error = amlt_sharded_last_error(nullptr);
        return st;
    }
    st = amlt_sharded_run(g, nullptr, task_source, dtype, ho, bounds, flags, nullptr, elapsed_s);
    g_sharded_error = st == AMLT_OK ? "" : g->err;
    amlt_sharded_destroy(g);
    return st;
}

const char* amlt_gpu_sharded_last_error(void) { return g_sharded_error.c_str(); }

}  // extern "C"
