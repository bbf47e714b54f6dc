// adapter_demo.cpp — the reference engine driving the B200 backend through
// integration/amlt_ref_gpu_backend.hpp, checked by the reference's OWN
// verifier (verify_against_naive, src/engine.cpp:186-210: exact on
// int-valued data, rel <= 1e-12 on real data).
//
// For each task (the reference's presets q1, q2, matmul, q3 and the sqdiff /
// eqcount statements) and each dims triple (the acceptance suite's dims,
// tests/acceptance.cpp:109-110, plus a larger one): compile_task,
// make_task_data (the reference's own seeded generator), run on the GPU via
// the adapter (run_adaptive and run_fixed), verify. A task the GPU has no
// body for (`A[i][k]*B[k][j] + u[i]*v[j]`) must raise UnsupportedExpression so
// the caller keeps the CPU path.
//
// Built by oracle/Makefile into oracle/_ref/ (it links the reference's
// objects); run by tests/test_gpu_integration.py on the GPU box.
//   adapter_demo            run + verify on cuda:0 (exit 0 iff all pass)
//   adapter_demo --dry-run  plumbing only (no device; nothing verified)
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "amlt/presets.hpp"
#include "amlt_ref_gpu_backend.hpp"

using namespace amlt;

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
                    if (fixed)
                        gpu::run_fixed(gpu, ct, data, bind, 64, 128, false, clock);
                    else
                        gpu::run_adaptive(gpu, ct, data, bind, false, clock);
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
    // a recognised MMLT the GPU has no body for: the adapter must refuse it
    bool refused = false;
    try {
        CompiledTask ct = compile_task(wrap_head + "A[i][k]*B[k][j] + u[i]*v[j];\n}\n", MachineModel{});
        DimBinding bind = bind_dims(ct, 8, 8, 8);
        TaskData data = make_task_data(ct, bind, 1, StorageOrder::RowMajor, StorageOrder::RowMajor,
                                       DataMode::IntValued);
        SteadyClock clock;
        if (dry)
            std::unique_ptr<amlt_gpu::Plan>(gpu::plan_for(gpu, ct));
        else
            gpu::run_adaptive(gpu, ct, data, bind, false, clock);
    } catch (const UnsupportedExpression&) {
        refused = true;
    } catch (const amlt_gpu::UnsupportedExpression&) {
        refused = true;
    }
    if (!refused) {
        ++failures;
        std::printf("FAIL a non-body MMLT was not refused\n");
    }
    std::printf("%s: %d checks, %d failures%s\n", failures ? "FAIL" : "PASS", checks, failures,
                dry ? " (dry run: plumbing only)" : "");
    return failures ? 1 : 0;
}
