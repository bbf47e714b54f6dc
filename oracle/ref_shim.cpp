// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// A thin extern "C" shim over the UNMODIFIED reference engine (amlt_core,
// compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// It exists so that tests/ and bench.py's reference arm can drive the
// reference's own entry points through ctypes:
//   compile_task      (reference src/engine.cpp:86-102)
//   bind_dims         (src/engine.cpp:104-126)
//   make_task_data    (src/engine.cpp:128-151; per-name seed seed^fnv1a(name))
//   run_naive         (src/naive.cpp:157-166; the declared correctness oracle)
//   run_adaptive      (src/engine.cpp:165-169 -> src/autotuner.cpp:103-151)
//   run_fixed         (src/engine.cpp:171-175 -> src/tiled_executor.cpp:9-77)
//   execute_scalar_region (src/kernel_exec.cpp:408-457)
//   gen_matrix / write_matrix_file / read_matrix_file (src/matrix.cpp:20-114)
//   adaptive_execute on row bands from N threads (the "all cores" CPU
//   baseline of SURVEY.md §8(d); each thread owns disjoint rows of R).
// Only tests/, __graft_entry__.smoke() and bench.py (cpu baseline / reference
// arm) load the resulting library. Nothing in paper_2305_08872_b200/ links it.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "amlt/clock.hpp"
#include "amlt/engine.hpp"
#include "amlt/errors.hpp"
#include "amlt/matrix.hpp"
#include "amlt/presets.hpp"
#include "amlt/schedule.hpp"

using namespace amlt;

namespace {

thread_local std::string g_err;

struct RefTask {
    CompiledTask ct;
    DimBinding bind;
    TaskData data;
    std::vector<std::string> names;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const UnsupportedExpression& e) {
        g_err = e.what();
        return 2;
    } catch (const MissingBinding& e) {
        g_err = e.what();
        return 3;
    } catch (const EngineError& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Copies the preset's DSL text into buf; returns its length or -1 if unknown.
int ref_preset_source(const char* name, char* buf, int buflen) {
    auto src = preset_source(name);
    if (!src) return -1;
    int n = static_cast<int>(src->size());
    if (buf && buflen > 0) {
        int c = std::min(n, buflen - 1);
        std::memcpy(buf, src->data(), static_cast<size_t>(c));
        buf[c] = 0;
    }
    return n;
}

void* ref_task_new(const char* src, std::int64_t M, std::int64_t K, std::int64_t N,
                   std::uint64_t seed, int order_a, int order_b, int int_valued) {
    RefTask* t = new RefTask();
    int rc = guarded([&] {
        t->ct = compile_task(src, MachineModel{});
        t->bind = bind_dims(t->ct, M, K, N);
        t->data = make_task_data(t->ct, t->bind, seed, static_cast<StorageOrder>(order_a),
                                 static_cast<StorageOrder>(order_b),
                                 int_valued ? DataMode::IntValued : DataMode::Real);
        for (const auto& kv : t->data.arrays) t->names.push_back(kv.first);
    });
    if (rc != 0) {
        delete t;
        return nullptr;
    }
    return t;
}

void ref_task_free(void* h) { delete static_cast<RefTask*>(h); }

int ref_task_is_mmlt(void* h) { return static_cast<RefTask*>(h)->ct.mmlt ? 1 : 0; }

// The reference's compiled pseudo-program (schedule_labelfs over the task's
// DAG, print_program: one "opcode dst src..." per line); returns its length.
int ref_task_program(void* h, char* buf, int buflen) {
    const RefTask* t = static_cast<RefTask*>(h);
    if (!t->ct.mmlt) return -1;
    const std::string s = print_program(schedule_labelfs(t->ct.dag));
    if (buf && buflen > 0) {
        std::strncpy(buf, s.c_str(), static_cast<size_t>(buflen - 1));
        buf[buflen - 1] = 0;
    }
    return static_cast<int>(s.size());
}

int ref_task_num_arrays(void* h) { return static_cast<int>(static_cast<RefTask*>(h)->names.size()); }

const char* ref_task_array_name(void* h, int idx) {
    return static_cast<RefTask*>(h)->names.at(static_cast<size_t>(idx)).c_str();
}

const char* ref_task_result_name(void* h) {
    return static_cast<RefTask*>(h)->data.result_name.c_str();
}

// Kernel footprint chosen by the reference planner (i_h, i_w).
void ref_task_shape(void* h, int* ih, int* iw) {
    auto* t = static_cast<RefTask*>(h);
    *ih = t->ct.plan.shape.i_h;
    *iw = t->ct.plan.shape.i_w;
}

// Role names for a recognised task: A, B and the aux leaf names (comma list).
int ref_task_roles(void* h, char* a, char* b, char* aux, int buflen) {
    auto* t = static_cast<RefTask*>(h);
    if (!t->ct.mmlt) return -1;
    std::snprintf(a, static_cast<size_t>(buflen), "%s", t->ct.recog.a.c_str());
    std::snprintf(b, static_cast<size_t>(buflen), "%s", t->ct.recog.b.c_str());
    std::string s;
    for (const auto& l : t->ct.recog.aux) {
        if (!s.empty()) s += ",";
        s += l.name;
    }
    std::snprintf(aux, static_cast<size_t>(buflen), "%s", s.c_str());
    return 0;
}

int ref_task_array_shape(void* h, const char* name, std::int64_t* rows, std::int64_t* cols,
                         int* order) {
    auto* t = static_cast<RefTask*>(h);
    auto it = t->data.arrays.find(name);
    if (it == t->data.arrays.end()) return -1;
    *rows = it->second.rows();
    *cols = it->second.cols();
    *order = static_cast<int>(it->second.order());
    return 0;
}

// Copies the array out in its STORAGE order (rows*cols doubles).
int ref_task_array_get(void* h, const char* name, double* out) {
    auto* t = static_cast<RefTask*>(h);
    auto it = t->data.arrays.find(name);
    if (it == t->data.arrays.end()) return -1;
    const MatrixBuffer& m = it->second;
    std::memcpy(out, m.data(), sizeof(double) * static_cast<size_t>(m.rows() * m.cols()));
    return 0;
}

int ref_task_array_set(void* h, const char* name, const double* in) {
    auto* t = static_cast<RefTask*>(h);
    auto it = t->data.arrays.find(name);
    if (it == t->data.arrays.end()) return -1;
    MatrixBuffer& m = it->second;
    std::memcpy(m.data(), in, sizeof(double) * static_cast<size_t>(m.rows() * m.cols()));
    return 0;
}

void ref_task_bounds(void* h, std::int64_t* out6) {
    const Bounds& b = static_cast<RefTask*>(h)->bind.bounds;
    out6[0] = b.i0; out6[1] = b.i1; out6[2] = b.j0; out6[3] = b.j1; out6[4] = b.k0; out6[5] = b.k1;
}

// run_naive over the task's own data (R updated in place).
int ref_task_run_naive(void* h, double* seconds) {
    auto* t = static_cast<RefTask*>(h);
    return guarded([&] { *seconds = run_naive_task(t->ct, t->data, t->bind); });
}

int ref_task_run_adaptive(void* h, int pack, double* seconds, std::int64_t* best_kc,
                          std::int64_t* best_nc) {
    auto* t = static_cast<RefTask*>(h);
    return guarded([&] {
        SteadyClock clock;
        TuneReport rep = run_adaptive(t->ct, t->data, t->bind, pack != 0, clock);
        *seconds = rep.total_seconds;
        if (best_kc) *best_kc = rep.best_kc;
        if (best_nc) *best_nc = rep.best_nc;
    });
}

// run_adaptive driven by the reference's FakeClock (clock.hpp:29-55) with the
// given interval script: the tuner's decisions and the number of intervals it
// consumed, for comparing tuner logic decision-for-decision.
int ref_task_run_adaptive_scripted(void* h, const double* deltas, int n, std::int64_t* best_kc,
                                   std::int64_t* best_nc, int* tuned, int* consumed,
                                   int* n_cover, std::int64_t* cover4) {
    auto* t = static_cast<RefTask*>(h);
    return guarded([&] {
        FakeClock clock(std::vector<double>(deltas, deltas + n));
        TuneReport rep = run_adaptive(t->ct, t->data, t->bind, false, clock);
        *best_kc = rep.best_kc;
        *best_nc = rep.best_nc;
        *tuned = rep.tuned ? 1 : 0;
        *consumed = static_cast<int>(clock.consumed());
        int m = 0;
        for (const auto& c : rep.coverage) {
            if (m >= *n_cover) break;
            cover4[4 * m + 0] = c.k0;
            cover4[4 * m + 1] = c.k1;
            cover4[4 * m + 2] = c.j0;
            cover4[4 * m + 3] = c.j1;
            ++m;
        }
        *n_cover = m;
    });
}

int ref_task_run_fixed(void* h, std::int64_t kc, std::int64_t nc, int pack, double* seconds) {
    auto* t = static_cast<RefTask*>(h);
    return guarded([&] {
        SteadyClock clock;
        *seconds = run_fixed(t->ct, t->data, t->bind, kc, nc, pack != 0, clock);
    });
}

int ref_task_run_scalar_region(void* h, std::int64_t i0, std::int64_t i1, std::int64_t j0,
                               std::int64_t j1, std::int64_t k0, std::int64_t k1) {
    auto* t = static_cast<RefTask*>(h);
    return guarded([&] {
        Operands ops = make_operands(t->ct, t->data);
        execute_scalar_region(t->ct.plan, t->ct.kernel, ops, i0, i1, j0, j1, k0, k1);
    });
}

// The reference's own adaptive executor on nthreads disjoint row bands of the
// rectangle [i0,i1) x [j0,j1) x full K, one std::thread each, timed by wall
// clock around the whole fan-out (steady_clock). Rows of R are independent, so
// the result equals the single-thread run bit for bit on int-valued data.
int ref_task_run_adaptive_bands(void* h, int nthreads, std::int64_t i0, std::int64_t i1,
                                std::int64_t j0, std::int64_t j1, double* seconds) {
    auto* t = static_cast<RefTask*>(h);
    return guarded([&] {
        Operands ops = make_operands(t->ct, t->data);
        const Bounds full = t->bind.bounds;
        const std::int64_t rows = i1 - i0;
        int nt = std::max(1, std::min<int>(nthreads, static_cast<int>(std::max<std::int64_t>(rows, 1))));
        std::vector<std::thread> th;
        std::vector<std::string> errs(static_cast<size_t>(nt));
        auto t0 = std::chrono::steady_clock::now();
        for (int w = 0; w < nt; ++w) {
            std::int64_t r0 = i0 + rows * w / nt, r1 = i0 + rows * (w + 1) / nt;
            th.emplace_back([&, w, r0, r1] {
                try {
                    SteadyClock clock;
                    Bounds b{r0, r1, j0, j1, full.k0, full.k1};
                    adaptive_execute(t->ct.plan, t->ct.kernel, ops, b, false, clock);
                } catch (const std::exception& e) {
                    errs[static_cast<size_t>(w)] = e.what();
                }
            });
        }
        for (auto& x : th) x.join();
        auto t1 = std::chrono::steady_clock::now();
        for (auto& e : errs)
            if (!e.empty()) throw EngineError(e);
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// gen_matrix (src/matrix.cpp:20-37): values in storage order into out.
int ref_gen_matrix(std::uint64_t seed, std::int64_t rows, std::int64_t cols, int order, int mode,
                   double* out) {
    return guarded([&] {
        MatrixBuffer m = gen_matrix(seed, rows, cols, static_cast<StorageOrder>(order),
                                    mode == 0 ? DataMode::IntValued : DataMode::Real);
        std::memcpy(out, m.data(), static_cast<size_t>(rows * cols) * sizeof(double));
    });
}

// write_matrix_file (src/matrix.cpp:64-88) of a storage-order buffer.
int ref_write_matrix_file(const char* path, std::int64_t rows, std::int64_t cols, int order,
                          const double* data) {
    return guarded([&] {
        MatrixBuffer m(rows, cols, static_cast<StorageOrder>(order));
        std::memcpy(m.data(), data, static_cast<size_t>(rows * cols) * sizeof(double));
        write_matrix_file(path, m);
    });
}

// read_matrix_file (src/matrix.cpp:90-114). out may be null (header only);
// otherwise it must hold cap doubles.
int ref_read_matrix_file(const char* path, std::int64_t* rows, std::int64_t* cols, int* order,
                         double* out, std::int64_t cap) {
    return guarded([&] {
        MatrixBuffer m = read_matrix_file(path);
        *rows = m.rows();
        *cols = m.cols();
        *order = static_cast<int>(m.order());
        const std::int64_t n = m.rows() * m.cols();
        if (out) {
            if (n > cap) throw EngineError("buffer too small");
            std::memcpy(out, m.data(), static_cast<size_t>(n) * sizeof(double));
        }
    });
}

}  // extern "C"
