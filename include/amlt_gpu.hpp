// amlt_gpu.hpp — header-only C++ host layer over the C-ABI (amlt_gpu.h).
//
// Mirrors the reference engine's C++ call shapes so a caller of
//   amlt::run_subtask      (include/amlt/tiled_executor.hpp:42-44)
//   amlt::adaptive_execute (include/amlt/autotuner.hpp:68-70)
//   amlt::compile_task     (include/amlt/engine.hpp:30-40)
// swaps to the B200 backend with the same argument meaning and the same
// error behaviour: C status codes are rethrown as the matching EngineError
// subclass (include/amlt/errors.hpp:10-60), and time flows through the same
// Clock seam (include/amlt/clock.hpp:12-55; FakeClock semantics included).
#pragma once

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "amlt_gpu.h"

namespace amlt_gpu {

// ---------------------------------------------------------------------------
// errors (errors.hpp:10-60)

class EngineError : public std::runtime_error {
public:
    explicit EngineError(const std::string& m) : std::runtime_error(m) {}
};
class UnsupportedExpression : public EngineError {
public:
    using EngineError::EngineError;
};
class MissingBinding : public EngineError {
public:
    using EngineError::EngineError;
};
class NoFeasibleKernel : public EngineError {
public:
    using EngineError::EngineError;
};
class NonPositiveTime : public EngineError {
public:
    using EngineError::EngineError;
};
class CudaError : public EngineError {
public:
    using EngineError::EngineError;
};
class NoDevice : public EngineError {
public:
    using EngineError::EngineError;
};

inline void check(amlt_status st, const amlt_ctx* ctx) {
    if (st == AMLT_OK) return;
    std::string m = amlt_gpu_last_error(ctx);
    switch (st) {
        case AMLT_ERR_UNSUPPORTED: throw UnsupportedExpression(m);
        case AMLT_ERR_MISSING_BINDING: throw MissingBinding(m);
        case AMLT_ERR_NO_FEASIBLE_KERNEL: throw NoFeasibleKernel(m);
        case AMLT_ERR_NON_POSITIVE_TIME: throw NonPositiveTime(m);
        case AMLT_ERR_CUDA: throw CudaError(m);
        case AMLT_ERR_NO_DEVICE: throw NoDevice(m);
        default: throw EngineError(m);
    }
}

// ---------------------------------------------------------------------------
// clock seam (clock.hpp:12-55)

class Clock {
public:
    virtual ~Clock() = default;
    virtual double now() = 0;
    static double thunk(void* self) { return static_cast<Clock*>(self)->now(); }
};

class SteadyClock final : public Clock {
public:
    double now() override {
        return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
            .count();
    }
};

// Scripted: now() alternates interval start / end; each completed interval
// advances by the next delta; throws when the script runs out.
class FakeClock final : public Clock {
public:
    FakeClock() = default;
    explicit FakeClock(std::vector<double> d) : deltas_(std::move(d)) {}
    void push(double d) { deltas_.push_back(d); }
    double now() override {
        if (!open_) {
            open_ = true;
            return t_;
        }
        open_ = false;
        if (next_ >= deltas_.size()) throw std::out_of_range("FakeClock: delta script exhausted");
        t_ += deltas_[next_++];
        return t_;
    }
    std::size_t consumed() const { return next_; }

private:
    std::vector<double> deltas_;
    std::size_t next_ = 0;
    double t_ = 0.0;
    bool open_ = false;
};

// ---------------------------------------------------------------------------
// plain records (tiled_executor.hpp:11-34, autotuner.hpp:11-34)

struct TileParams {
    std::int64_t kc = 0;
    std::int64_t nc = 0;
    bool pack = false;
    int variant = -1;
};
using Bounds = amlt_bounds;
using ExecRecord = amlt_exec_record;
struct ExecLog {
    std::vector<ExecRecord> records;
};
using Trial = amlt_trial;
using CoverRect = amlt_cover_rect;
struct TuneReport {
    std::vector<Trial> trials;
    int best_variant = -1;
    std::int64_t best_kc = 0;
    bool tuned = false;
    bool from_cache = false;
    bool scratch_tuned = false;
    std::vector<CoverRect> coverage;
    double tuning_fraction = 0.0;
    double total_seconds = 0.0;
    double tuning_seconds = 0.0;  // scratch (whole-task) trials, included in total_seconds
    int refined = 0;              // > 0: the winner is the best of the last `refined` (8-wave) trials
};

// A MatrixBuffer-like view (device memory for run_subtask / adaptive_execute,
// host memory for run_host).
struct Matrix {
    void* data = nullptr;
    std::int64_t rows = 0, cols = 0, ld = 0;
    amlt_order order = AMLT_ROW_MAJOR;
    amlt_dtype dtype = AMLT_F64;
    amlt_matrix c() const { return amlt_matrix{data, rows, cols, ld, order, dtype}; }
};

struct Operands {
    Matrix a, b, r, thres, dis;
    int n_aux = 0;              // generated bodies: aux leaves by position
    Matrix aux[AMLT_MAX_AUX];   // (Plan::roles().aux_names)
    amlt_operands c() const {
        amlt_operands o{};
        o.a = a.c();
        o.b = b.c();
        o.r = r.c();
        o.thres = thres.c();
        o.dis = dis.c();
        o.n_aux = n_aux;
        for (int q = 0; q < n_aux && q < AMLT_MAX_AUX; ++q) o.aux[q] = aux[q].c();
        return o;
    }
};

// ---------------------------------------------------------------------------
// context + plan (RAII)

class Context {
public:
    explicit Context(int device = 0, bool dry_run = false) {
        check(amlt_gpu_ctx_create(device, dry_run ? AMLT_CTX_DRY_RUN : 0, &ctx_), nullptr);
    }
    ~Context() { amlt_gpu_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    amlt_ctx* get() const { return ctx_; }
    void set_stream(void* cuda_stream) { check(amlt_gpu_set_stream(ctx_, cuda_stream), ctx_); }

private:
    amlt_ctx* ctx_ = nullptr;
};

// A device matrix owned by the library's allocator (amlt_gpu_matrix_*):
// f64 values in, stored in the plan's dtype, f64 values out.
class DeviceMatrix {
public:
    DeviceMatrix(Context& ctx, std::int64_t rows, std::int64_t cols, amlt_order order,
                 amlt_dtype dtype)
        : ctx_(&ctx) {
        check(amlt_gpu_matrix_alloc(ctx.get(), rows, cols, order, dtype, &m_), ctx.get());
    }
    ~DeviceMatrix() { amlt_gpu_matrix_free(ctx_->get(), &m_); }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
    void upload(const double* host, std::int64_t host_ld) {
        check(amlt_gpu_matrix_upload(ctx_->get(), &m_, host, host_ld), ctx_->get());
    }
    void download(double* host, std::int64_t host_ld) const {
        check(amlt_gpu_matrix_download(ctx_->get(), &m_, host, host_ld), ctx_->get());
    }
    Matrix view() const {
        Matrix v;
        v.data = m_.data;
        v.rows = m_.rows;
        v.cols = m_.cols;
        v.ld = m_.ld;
        v.order = static_cast<amlt_order>(m_.order);
        v.dtype = static_cast<amlt_dtype>(m_.dtype);
        return v;
    }

private:
    Context* ctx_;
    amlt_matrix m_{};
};

// The GPU counterpart of CompiledTask: immutable, shareable.
class Plan {
public:
    Plan(Context& ctx, const amlt_body_desc& d) : ctx_(&ctx) {
        check(amlt_gpu_plan_create(ctx.get(), &d, &plan_), ctx.get());
    }
    // compile_task(source) for the GPU bodies; UnsupportedExpression otherwise
    Plan(Context& ctx, const std::string& task_source, amlt_dtype dtype) : ctx_(&ctx) {
        check(amlt_gpu_plan_from_source(ctx.get(), task_source.c_str(), dtype, &plan_, &info_),
              ctx.get());
    }
    ~Plan() { amlt_gpu_plan_destroy(plan_); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    const amlt_plan* get() const { return plan_; }
    Context& ctx() const { return *ctx_; }
    const amlt_task_info& roles() const { return info_; }
    int num_variants() const { return amlt_gpu_plan_num_variants(plan_); }
    amlt_variant_info variant(int idx) const {
        amlt_variant_info v{};
        check(amlt_gpu_plan_variant(plan_, idx, &v), ctx_->get());
        return v;
    }

private:
    Context* ctx_;
    amlt_plan* plan_ = nullptr;
    amlt_task_info info_{};
};

// ---------------------------------------------------------------------------
// executors

namespace detail {
struct LogBuf {
    explicit LogBuf(ExecLog* l) : log(l) {
        if (log) {
            recs.resize(4096);
            c = amlt_exec_log{recs.data(), static_cast<int32_t>(recs.size()), 0, 0};
        }
    }
    amlt_exec_log* ptr() { return log ? &c : nullptr; }
    void flush() {
        if (log) log->records.insert(log->records.end(), recs.begin(), recs.begin() + c.count);
    }
    ExecLog* log;
    std::vector<ExecRecord> recs;
    amlt_exec_log c{};
};
inline amlt_tile_params tile(const TileParams& t) {
    return amlt_tile_params{t.kc, t.nc, t.pack ? 1 : 0, t.variant};
}
}  // namespace detail

// run_subtask (tiled_executor.hpp:42-44): elapsed seconds between the two
// clock reads around the synchronous GPU work.
inline double run_subtask(const Plan& plan, const Operands& ops, const TileParams& params,
                          const Bounds& b, Clock& clock, ExecLog* log = nullptr) {
    amlt_operands o = ops.c();
    amlt_tile_params t = detail::tile(params);
    detail::LogBuf lb(log);
    double el = 0;
    check(amlt_gpu_run_subtask(plan.ctx().get(), plan.get(), &o, &t, &b, &Clock::thunk, &clock,
                               lb.ptr(), &el),
          plan.ctx().get());
    lb.flush();
    return el;
}

// adaptive_execute (autotuner.hpp:68-70).
inline TuneReport adaptive_execute(const Plan& plan, const Operands& ops, const Bounds& b,
                                   bool pack, Clock& clock, ExecLog* log = nullptr) {
    amlt_operands o = ops.c();
    amlt_tune_report r{};
    detail::LogBuf lb(log);
    check(amlt_gpu_adaptive_execute(plan.ctx().get(), plan.get(), &o, &b, pack ? 1 : 0,
                                    &Clock::thunk, &clock, lb.ptr(), &r),
          plan.ctx().get());
    lb.flush();
    TuneReport rep;
    rep.trials.assign(r.trials, r.trials + r.n_trials);
    rep.best_variant = r.best_variant;
    rep.best_kc = r.best_kc;
    rep.tuned = r.tuned != 0;
    rep.from_cache = r.from_cache != 0;
    rep.scratch_tuned = r.scratch_tuned != 0;
    rep.coverage.assign(r.coverage, r.coverage + r.n_cover);
    rep.tuning_fraction = r.tuning_fraction;
    rep.total_seconds = r.total_seconds;
    rep.tuning_seconds = r.tuning_seconds;
    rep.refined = r.refined;
    return rep;
}

namespace detail {
inline TuneReport report_of(const amlt_tune_report& r) {
    TuneReport rep;
    rep.trials.assign(r.trials, r.trials + r.n_trials);
    rep.best_variant = r.best_variant;
    rep.best_kc = r.best_kc;
    rep.tuned = r.tuned != 0;
    rep.from_cache = r.from_cache != 0;
    rep.scratch_tuned = r.scratch_tuned != 0;
    rep.coverage.assign(r.coverage, r.coverage + r.n_cover);
    rep.tuning_fraction = r.tuning_fraction;
    rep.total_seconds = r.total_seconds;
    rep.tuning_seconds = r.tuning_seconds;
    rep.refined = r.refined;
    return rep;
}
}  // namespace detail

// run_adaptive over host MatrixBuffers (amlt_gpu_run_host_adaptive): tunes
// on the first call of a shape, reuses the winner after; the report's
// total_seconds covers the copies too.
inline TuneReport run_host_adaptive(const Plan& plan, const Operands& host_ops, const Bounds& b,
                                    Clock& clock, bool r_zero = false) {
    amlt_operands o = host_ops.c();
    amlt_tune_report r{};
    double el = 0;
    check(amlt_gpu_run_host_adaptive(plan.ctx().get(), plan.get(), &o, &b, r_zero ? AMLT_HOST_R_ZERO : 0,
                                     &Clock::thunk, &clock, &r, &el),
          plan.ctx().get());
    return detail::report_of(r);
}

// Host MatrixBuffers in, host R out (copies + compute inside the interval).
inline double run_host(const Plan& plan, const Operands& host_ops, const Bounds& b, Clock& clock,
                       const TileParams* params = nullptr, bool r_zero = false) {
    amlt_operands o = host_ops.c();
    amlt_tile_params t{};
    if (params) t = detail::tile(*params);
    double el = 0;
    check(amlt_gpu_run_host(plan.ctx().get(), plan.get(), &o, params ? &t : nullptr, &b,
                            r_zero ? AMLT_HOST_R_ZERO : 0, &Clock::thunk, &clock, &el),
          plan.ctx().get());
    return el;
}

// spr (engine.hpp:83-85).
inline double spr(std::int64_t M, std::int64_t K, std::int64_t N, double seconds) {
    double out = 0;
    amlt_status st = amlt_spr(M, K, N, seconds, &out);
    if (st == AMLT_ERR_NON_POSITIVE_TIME)
        throw NonPositiveTime("elapsed time must be positive, got " + std::to_string(seconds));
    check(st, nullptr);
    return out;
}

}  // namespace amlt_gpu
