// amlt_ref_gpu_backend.hpp — the file a maintainer of the reference engine
// (/root/reference/proj, "amlt") adds to route its MMLT executor to the B200
// backend. It is written against the reference's public headers and this
// repo's C-ABI (include/amlt_gpu.h via the C++ layer include/amlt_gpu.hpp):
//
//   amlt::run_adaptive(ct, data, bind, pack, clock, log)        engine.hpp:65-66
//   amlt::run_fixed(ct, data, bind, kc, nc, pack, clock, log)   engine.hpp:67-68
//
// become
//
//   amlt::gpu::run_adaptive(gpu, ct, data, bind, pack, clock)
//   amlt::gpu::run_fixed(gpu, ct, data, bind, kc, nc, pack, clock)
//
// with the same arguments, the same Clock (the reference's FakeClock drives
// the GPU executor's timing too), the same result in data.result(), and the
// same errors (UnsupportedExpression for a task that is not
// multiply-accumulate-like, so the caller keeps its CPU path for it; every
// recognised statement runs on the GPU, the six fixed bodies through their
// hand-written kernels and the rest through bodies generated at plan time). Operands stay the reference's
// f64 MatrixBuffers in host memory; the backend copies them in and R out.
#pragma once

#include <algorithm>
#include <memory>
#include <string>

#include "amlt/ast.hpp"
#include "amlt/autotuner.hpp"
#include "amlt/clock.hpp"
#include "amlt/engine.hpp"
#include "amlt/errors.hpp"
#include "amlt_gpu.hpp"

namespace amlt::gpu {

// The reference Clock drives the GPU executor's clock seam.
class ClockBridge final : public amlt_gpu::Clock {
public:
    explicit ClockBridge(amlt::Clock& c) : c_(c) {}
    double now() override { return c_.now(); }

private:
    amlt::Clock& c_;
};

inline amlt_gpu::Matrix view(const MatrixBuffer& m) {
    amlt_gpu::Matrix v;
    v.data = const_cast<double*>(m.data());
    v.rows = m.rows();
    v.cols = m.cols();
    v.ld = m.stride();
    v.order = m.order() == StorageOrder::RowMajor ? AMLT_ROW_MAJOR : AMLT_COL_MAJOR;
    v.dtype = AMLT_F64;
    return v;
}

// make_operands (engine.cpp:153-163) for the GPU: roles by the recogniser's
// names; a missing aux array raises MissingBinding like the reference.
inline amlt_gpu::Operands operands(const amlt_gpu::Plan& plan, TaskData& data) {
    const amlt_task_info& r = plan.roles();
    auto need = [&](const char* name) -> MatrixBuffer& {
        auto it = data.arrays.find(name);
        if (it == data.arrays.end()) throw MissingBinding(name);
        return it->second;
    };
    amlt_gpu::Operands ops;
    ops.a = view(need(r.a));
    ops.b = view(need(r.b));
    ops.r = view(data.result());
    if (r.thres[0]) ops.thres = view(need(r.thres));
    if (r.dis[0]) ops.dis = view(need(r.dis));
    // generated bodies (any other recognised statement): aux leaves by position
    ops.n_aux = r.n_aux;
    for (int q = 0; q < r.n_aux; ++q) ops.aux[q] = view(need(r.aux_names[q]));
    return ops;
}

// compile_task for the GPU; the reference's own canonical text of the task
// (print_task, ast.hpp:73) is what the backend recognises.
inline amlt_gpu::Plan* plan_for(amlt_gpu::Context& gpu, const CompiledTask& ct) {
    try {
        return new amlt_gpu::Plan(gpu, print_task(ct.task), AMLT_F64);
    } catch (const amlt_gpu::UnsupportedExpression& e) {
        throw UnsupportedExpression(e.what());
    }
}

inline Bounds to_ref(const amlt_bounds& b) { return Bounds{b.i0, b.i1, b.j0, b.j1, b.k0, b.k1}; }
inline amlt_bounds to_gpu(const Bounds& b) { return amlt_bounds{b.i0, b.i1, b.j0, b.j1, b.k0, b.k1}; }

// run_fixed: one subtask over the whole bounds with TileParams{kc, nc}.
inline double run_fixed(amlt_gpu::Context& gpu, const CompiledTask& ct, TaskData& data,
                        const DimBinding& bind, std::int64_t kc, std::int64_t nc, bool pack,
                        amlt::Clock& clock) {
    std::unique_ptr<amlt_gpu::Plan> plan(plan_for(gpu, ct));
    amlt_gpu::Operands ops = operands(*plan, data);
    amlt_gpu::TileParams tp;
    tp.kc = kc;
    tp.nc = nc;
    tp.pack = pack;
    ClockBridge cb(clock);
    return amlt_gpu::run_host(*plan, ops, to_gpu(bind.bounds), cb, &tp);
}

// run_adaptive: the GPU runtime tuner over host buffers
// (amlt_gpu_run_host_adaptive), its report mapped onto the reference
// TuneReport (autotuner.hpp:11-34) without inventing anything:
//   tuned         true iff this call measured candidates (row-band or
//                 scratch trials); false when the winner came from an earlier
//                 call of the same shape (no trials then) or the task ran
//                 untuned
//   nc_trials     one per tile variant measured: value = the variant's CTA
//                 width (the GPU planner's nc, amlt_tile_params.nc), elapsed
//                 = its measured seconds, score = seconds per output row of
//                 its band (the GPU tuner lays candidates on row bands; lower
//                 is better, as the reference's elapsed/nc)
//   kc_trials     empty: the GPU tuner does not search kc on these sizes
//   best_kc       the winner's K-segment depth (K when it runs whole K)
//   best_nc       the winner's CTA width
//   coverage      the (k, j) rectangles completed for ALL rows: the GPU
//                 report's row-band rectangles are checked to tile
//                 [i0, i1) x (k, j) exactly once and merged over rows, so the
//                 reference's invariant holds (pairwise disjoint, union K x N)
//   tuning_fraction  rows measured by trials / M (the GPU tuner's unit)
//   total_seconds    all subtasks and copies
// The reference's own kc / nc search (find_kc, find_nc) stays available
// on the GPU as amlt_gpu_adaptive_execute_amulet.
inline TuneReport run_adaptive(amlt_gpu::Context& gpu, const CompiledTask& ct, TaskData& data,
                               const DimBinding& bind, bool pack, amlt::Clock& clock) {
    std::unique_ptr<amlt_gpu::Plan> plan(plan_for(gpu, ct));
    amlt_gpu::Operands ops = operands(*plan, data);
    ClockBridge cb(clock);
    (void)pack;  // operands are always staged through shared memory
    const amlt_bounds gb = to_gpu(bind.bounds);
    amlt_gpu::TuneReport g = amlt_gpu::run_host_adaptive(*plan, ops, gb, cb);
    TuneReport rep;
    rep.tuned = g.tuned || g.scratch_tuned;
    for (const amlt_trial& t : g.trials)
        rep.nc_trials.push_back(Trial{plan->variant(static_cast<int>(t.value)).block_n, t.elapsed, t.score});
    rep.best_kc = g.best_kc;
    rep.best_nc = g.best_variant >= 0 ? plan->variant(g.best_variant).block_n : gb.j1 - gb.j0;
    // merge the row bands of each (k, j) rectangle; each must tile the rows once
    std::vector<std::pair<CoverRect, std::int64_t>> kj;  // rect, rows covered
    for (const amlt_cover_rect& c : g.coverage) {
        auto it = std::find_if(kj.begin(), kj.end(), [&](const auto& e) {
            return e.first.k0 == c.k0 && e.first.k1 == c.k1 && e.first.j0 == c.j0 && e.first.j1 == c.j1;
        });
        if (it == kj.end()) kj.push_back({CoverRect{c.k0, c.k1, c.j0, c.j1}, c.i1 - c.i0});
        else it->second += c.i1 - c.i0;
    }
    for (const auto& e : kj) {
        if (e.second != gb.i1 - gb.i0)
            throw EngineError("GPU coverage does not tile the rows of a (k, j) rectangle exactly once");
        rep.coverage.push_back(e.first);
    }
    rep.tuning_fraction = g.tuning_fraction;
    rep.total_seconds = g.total_seconds;
    return rep;
}

}  // namespace amlt::gpu
