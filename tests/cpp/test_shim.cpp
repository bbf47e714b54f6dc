// C++ host layer (include/amlt_gpu.hpp) over the C-ABI, in a dry-run
// context: the reference's call shapes, Clock seam and error mapping.
// Built and run by tests/test_integration.py (no GPU needed).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "amlt_gpu.hpp"

#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::printf("CHECK failed line %d: %s\n", __LINE__, #c);          \
            std::exit(1);                                                     \
        }                                                                     \
    } while (0)

int main() {
    using namespace amlt_gpu;
    Context ctx(0, /*dry_run=*/true);
    const char* q1 =
        "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n"
        "  R[i][j] += A[i][k]*B[k][j] - (A[i][k]*B[k][j] > thres[j])*A[i][k]*B[k][j]*dis[j];\n}\n";
    Plan plan(ctx, q1, AMLT_F64);
    CHECK(plan.roles().desc.body == AMLT_BODY_DISCOUNT);
    CHECK(std::string(plan.roles().thres) == "thres" && std::string(plan.roles().dis) == "dis");

    const std::int64_t M = 131072, K = 64, N = 1024;
    // dry-run: buffers are described, never touched
    std::vector<double> tiny(16);
    auto mat = [&](std::int64_t r, std::int64_t c) {
        Matrix m;
        m.data = reinterpret_cast<void*>(0x10000);  // never dereferenced in dry-run
        m.rows = r;
        m.cols = c;
        m.ld = c;
        return m;
    };
    Operands ops;
    ops.a = mat(M, K);
    ops.b = mat(K, N);
    ops.r = mat(M, N);
    ops.thres = mat(N, 1);
    ops.dis = mat(N, 1);

    // run_subtask reads the clock exactly twice
    FakeClock fc({0.5});
    double el = run_subtask(plan, ops, TileParams{}, Bounds{0, 64, 0, 64, 0, K}, fc);
    CHECK(el == 0.5 && fc.consumed() == 1);

    // tuner: scripted intervals -> argmin(score) wins, rows covered once
    FakeClock tc({0.9, 0.2, 0.7, 0.8, 0.6, 0.4, 0.95, 0.85, 0.75, 0.65, 0.55, 0.45, 0.35, 0.99, 0.3, 0.25, 0.97, 0.96});
    ExecLog log;
    TuneReport rep = adaptive_execute(plan, ops, Bounds{0, M, 0, N, 0, K}, false, tc, &log);
    CHECK(rep.tuned && rep.trials.size() >= 2);
    std::size_t best = 0;
    for (std::size_t t = 1; t < rep.trials.size(); ++t)
        if (rep.trials[t].score < rep.trials[best].score) best = t;
    CHECK(rep.best_variant == rep.trials[best].value);
    CHECK(tc.consumed() == rep.trials.size() + 1);
    std::int64_t rows = 0;
    for (auto& c : rep.coverage) rows += c.i1 - c.i0;
    CHECK(rows == M && log.records.size() == rep.coverage.size());

    // errors map onto the reference hierarchy
    bool missing = false, unsupported = false, nonpos = false;
    Operands bad = ops;
    bad.dis = Matrix{};
    try {
        run_subtask(plan, bad, TileParams{}, Bounds{0, 8, 0, 8, 0, 8}, fc);
    } catch (const MissingBinding&) {
        missing = true;
    }
    try {
        Plan p2(ctx, "where(i in [0..M] and j in [0..N] and k in [0..K]) {\n  R[i][j] += A[i][k]*B[k][j]*u[k];\n}\n",
                AMLT_F64);
    } catch (const UnsupportedExpression&) {
        unsupported = true;
    }
    try {
        spr(1, 1, 1, 0.0);
    } catch (const NonPositiveTime&) {
        nonpos = true;
    }
    CHECK(missing && unsupported && nonpos);
    CHECK(spr(1000, 1000, 1000, 1.0) == 1.0);
    std::printf("PASS\n");
    return 0;
}
