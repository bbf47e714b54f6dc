// adapter_demo.cpp — the reference engine driving the B200 backend through
// integration/amlt_ref_gpu_backend.hpp, checked by the reference's OWN
// verifier (verify_against_naive, src/engine.cpp:186-210: exact on
// int-valued data, rel <= 1e-12 on real data).
//
// For each task (the reference's presets q1, q2, matmul, q3 and the sqdiff /
// eqcount statements) and each dims triple (the acceptance suite's dims,
// tests/acceptance.cpp:109-110, plus a larger one): compile_task,
// make_task_data (the reference's own seeded generator), run on the GPU via
// the adapter (run_adaptive and run_fixed), verify. Then random recognised
// statements outside the six bodies (aux leaves u[i], v[j], W[i][j], s,
// constants, + - * / and comparisons), which run through generated bodies.
// A statement that is not multiply-accumulate-like (`... * u[k]`) must
// raise UnsupportedExpression so the caller keeps the CPU path.
//
// Built by oracle/Makefile into oracle/_ref/ (it links the reference's
// objects); run by tests/test_gpu_integration.py on the GPU box.
//   adapter_demo            run + verify on cuda:0 (exit 0 iff all pass)
//   adapter_demo --dry-run  plumbing only (no device; nothing verified)
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "amlt/presets.hpp"
#include "amlt_ref_gpu_backend.hpp"

using namespace amlt;

// The reference's TuneReport invariants (autotuner.hpp:25-34): coverage
// pairwise disjoint with union K x N (checked cell by cell), trials present
// exactly when the call tuned, best_kc / best_nc inside the task.
bool report_ok(const TuneReport& rep, const Bounds& b) {
    const std::int64_t K = b.k1 - b.k0, N = b.j1 - b.j0;
    std::vector<int> cells(static_cast<size_t>(std::max<std::int64_t>(K * N, 0)), 0);
    for (const CoverRect& c : rep.coverage) {
        if (c.k0 < b.k0 || c.k1 > b.k1 || c.j0 < b.j0 || c.j1 > b.j1) return false;
        for (std::int64_t k = c.k0; k < c.k1; ++k)
            for (std::int64_t j = c.j0; j < c.j1; ++j) ++cells[static_cast<size_t>((k - b.k0) * N + (j - b.j0))];
    }
    for (int v : cells)
        if (v != 1) return false;
    if (rep.tuned != !rep.nc_trials.empty()) return false;
    if (rep.best_kc < 1 || rep.best_kc > std::max<std::int64_t>(K, 1) || rep.best_nc < 1) return false;
    return rep.total_seconds > 0;
}

int tuned_calls = 0;

int main(int argc, char** argv) {
    const bool dry = argc > 1 && std::strcmp(argv[1], "--dry-run") == 0;
    amlt_gpu::Context gpu(0, dry);
    const std::string wrap_head = "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] += ";
    std::vector<std::pair<std::string, std::string>> tasks = {
        {"q1", *preset_source("q1")},
        {"q2", *preset_source("q2")},
        {"matmul", *preset_source("matmul")},
        {"q3", *preset_source("q3")},
        {"q1-tc", *preset_source("q1-tc")},
        {"q1-ti", *preset_source("q1-ti")},
        {"q2-tij", *preset_source("q2-tij")},
        {"q3-ti", *preset_source("q3-ti")},
        {"matmul-atb", *preset_source("matmul-atb")},
        {"q1-tj-abt", *preset_source("q1-tj-abt")},
        {"q2-tij-atbt", *preset_source("q2-tij-atbt")},
        {"sqdiff", wrap_head + "(A[i][k] - B[k][j])*(A[i][k] - B[k][j]);\n}\n"},
        {"eqcount", wrap_head + "A[i][k] == B[k][j];\n}\n"},
    };
    const std::int64_t dims[][3] = {{64, 64, 64}, {96, 128, 160}, {257, 129, 65}, {13, 17, 5}};
    int failures = 0, checks = 0;
    for (const auto& [name, src] : tasks) {
        CompiledTask ct = compile_task(src, MachineModel{});
        for (const auto& d : dims) {
            for (DataMode mode : {DataMode::IntValued, DataMode::Real}) {
                if (mode == DataMode::Real && name == "eqcount") continue;  // counts of reals: trivially 0
                for (int fixed = 0; fixed < 2; ++fixed) {
                    DimBinding bind = bind_dims(ct, d[0], d[1], d[2]);
                    TaskData data = make_task_data(ct, bind, 1, StorageOrder::RowMajor,
                                                   StorageOrder::RowMajor, mode);
                    SteadyClock clock;
                    if (dry) {  // plumbing only: plan + operand mapping
                        std::unique_ptr<amlt_gpu::Plan> plan(gpu::plan_for(gpu, ct));
                        (void)gpu::operands(*plan, data);
                        continue;
                    }
                    if (fixed) {
                        gpu::run_fixed(gpu, ct, data, bind, 64, 128, false, clock);
                    } else {
                        TuneReport rep = gpu::run_adaptive(gpu, ct, data, bind, false, clock);
                        ++checks;
                        if (!report_ok(rep, bind.bounds)) {
                            ++failures;
                            std::printf("FAIL %s %lldx%lldx%lld: TuneReport invariants\n", name.c_str(),
                                        (long long)d[0], (long long)d[1], (long long)d[2]);
                        }
                        if (rep.tuned) ++tuned_calls;
                    }
                    VerifyResult v = verify_against_naive(ct, data, bind, mode);
                    ++checks;
                    if (!v.pass) {
                        ++failures;
                        std::printf("FAIL %s %s %lldx%lldx%lld %s: exact=%d max_rel=%.3e\n",
                                    name.c_str(), fixed ? "fixed" : "adaptive", (long long)d[0],
                                    (long long)d[1], (long long)d[2],
                                    mode == DataMode::IntValued ? "int" : "real", v.exact,
                                    v.max_rel_err);
                    }
                }
            }
        }
    }
    // every one of the reference's 52 presets at the dims of test_engine.cpp:145-167,
    // int-valued data, adaptive: bit-exact against run_naive
    const std::int64_t pdims[][3] = {{32, 24, 40}, {13, 17, 5}};
    for (const std::string& name : all_preset_names()) {
        CompiledTask ct = compile_task(*preset_source(name), MachineModel{});
        for (const auto& d : pdims) {
            DimBinding bind = bind_dims(ct, d[0], d[1], d[2]);
            TaskData data = make_task_data(ct, bind, 1, StorageOrder::RowMajor,
                                           StorageOrder::RowMajor, DataMode::IntValued);
            if (dry) {
                std::unique_ptr<amlt_gpu::Plan> plan(gpu::plan_for(gpu, ct));
                (void)gpu::operands(*plan, data);
                continue;
            }
            SteadyClock clock;
            gpu::run_adaptive(gpu, ct, data, bind, false, clock);
            VerifyResult v = verify_against_naive(ct, data, bind, DataMode::IntValued);
            ++checks;
            if (!v.exact) {
                ++failures;
                std::printf("FAIL preset %s %lldx%lldx%lld: max_abs=%.3e\n", name.c_str(),
                            (long long)d[0], (long long)d[1], (long long)d[2], v.max_abs_err);
            }
        }
    }
    // random recognised statements outside the six bodies: generated bodies
    // (compiled at plan time) must agree with run_naive bit for bit on
    // int-valued data, both orientations, row/col-major storage, "=" and "+="
    {
        std::mt19937_64 rng(20261020);
        auto pick = [&](int n) { return static_cast<int>(rng() % static_cast<unsigned>(n)); };
        const int n_stmt = dry ? 3 : 40;
        for (int n = 0; n < n_stmt; ++n) {
            const bool at = pick(3) == 0, bt = pick(3) == 0;
            const std::string A = at ? "A[k][i]" : "A[i][k]", B = bt ? "B[j][k]" : "B[k][j]";
            std::function<std::string(int)> expr = [&](int depth) -> std::string {
                if (depth >= 3 || pick(3) == 0) {
                    switch (pick(8)) {
                        case 0: return A;
                        case 1: return B;
                        case 2: return "u[i]";
                        case 3: return "v[j]";
                        case 4: return "W[i][j]";
                        case 5: return "s";
                        default: return std::to_string(pick(7));
                    }
                }
                const std::string l = expr(depth + 1);
                if (pick(10) == 0) return "(" + l + ")/" + std::to_string(2 << pick(3));
                static const char* ops[] = {" + ", " - ", "*", " > ", " >= ", " < ", " <= ", " == "};
                return "(" + l + ")" + ops[pick(pick(4) == 0 ? 8 : 3)] + "(" + expr(depth + 1) + ")";
            };
            const std::string rhs = A + "*" + B + (pick(2) ? " + " : " - ") + "(" + expr(0) + ")";
            const bool acc = pick(8) != 0;
            const std::string src = "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] " +
                                    std::string(acc ? "+=" : "=") + " " + rhs + ";\n}\n";
            CompiledTask ct = compile_task(src, MachineModel{});
            if (!ct.mmlt) continue;
            const std::int64_t M = 5 + pick(70), K = 1 + pick(60), N = 5 + pick(90);
            const StorageOrder oa = n % 2 ? StorageOrder::ColMajor : StorageOrder::RowMajor;
            const StorageOrder ob = n % 3 ? StorageOrder::ColMajor : StorageOrder::RowMajor;
            for (int fixed = 0; fixed < 2; ++fixed) {
                DimBinding bind = bind_dims(ct, M, K, N);
                TaskData data = make_task_data(ct, bind, 7 + n, oa, ob, DataMode::IntValued);
                if (dry) {
                    std::unique_ptr<amlt_gpu::Plan> plan(gpu::plan_for(gpu, ct));
                    (void)gpu::operands(*plan, data);
                    continue;
                }
                SteadyClock clock;
                if (fixed)
                    gpu::run_fixed(gpu, ct, data, bind, 32, 64, false, clock);
                else
                    gpu::run_adaptive(gpu, ct, data, bind, false, clock);
                VerifyResult v = verify_against_naive(ct, data, bind, DataMode::IntValued);
                ++checks;
                if (!v.exact) {
                    ++failures;
                    std::printf("FAIL generated %s %lldx%lldx%lld: max_abs=%.3e\n%s", fixed ? "fixed" : "adaptive",
                                (long long)M, (long long)K, (long long)N, v.max_abs_err, src.c_str());
                }
            }
        }
    }
    // a statement that is not multiply-accumulate-like: the adapter must refuse it
    bool refused = false;
    try {
        CompiledTask ct = compile_task(wrap_head + "A[i][k]*B[k][j]*u[k];\n}\n", MachineModel{});
        std::unique_ptr<amlt_gpu::Plan>(gpu::plan_for(gpu, ct));
    } catch (const UnsupportedExpression&) {
        refused = true;
    } catch (const amlt_gpu::UnsupportedExpression&) {
        refused = true;
    }
    if (!refused) {
        ++failures;
        std::printf("FAIL a non-MMLT statement was not refused\n");
    }
    // the fixed-body tasks above are small enough for whole-task trials: the
    // first call of each shape must have tuned
    if (!dry && tuned_calls == 0) {
        ++failures;
        std::printf("FAIL no run_adaptive call reported trials\n");
    }
    std::printf("%s: %d checks (%d tuned run_adaptive calls), %d failures%s\n", failures ? "FAIL" : "PASS",
                checks, tuned_calls, failures, dry ? " (dry run: plumbing only)" : "");
    return failures ? 1 : 0;
}
