/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement of the reference's correctness oracle for the MMLT hot
 * path: the naive interpreter `run_naive` (reference src/naive.cpp:157-166),
 * which walks the loop nest in declaration order i, j, k
 * (NaiveRunner::nest, src/naive.cpp:65-83) and evaluates the statement's
 * syntax tree in double precision for every (i, j, k)
 * (NaiveRunner::eval, src/naive.cpp:85-117), then does `R[i][j] += v`
 * (or `R[i][j] = v` for assignment statements, src/naive.cpp:73-76).
 *
 * The five bodies are the statements the reference builds for them
 * (presets src/presets.cpp:52-94, evaluated left-associatively as the
 * parser builds them, src/parser.cpp:142-365):
 *   GEMM      v = A*B                                         (preset matmul)
 *   DISCOUNT  v = A*B - (((A*B > T) * A) * B) * dis           (preset q1)
 *   BOOST     v = A*B + (A*B > T) * (A*B - T)                 (preset q2)
 *   SQDIFF    v = (A - B) * (A - B)
 *   EQCOUNT   v = (A == B)
 *   THRCOUNT  v = (A*B > T)                                   (preset q3)
 * Comparisons yield 1.0 / 0.0 (src/naive.cpp:108-112).
 *
 * Every operand is addressed through explicit (row, col) element strides so
 * one routine covers row-/col-major storage, the transposed orientations
 * (A[k][i], B[j][k]) and the threshold forms (-tc constant, -ti thres[i],
 * -tj thres[j], -tij thres[i][j]; stride 0 broadcasts).
 *
 * Compile with -ffp-contract=off: each C operator below is one IEEE double
 * operation, exactly as the tree walker performs it.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use
 * this file; the product path (paper_2305_08872_b200/) never does.
 */
#include <stdint.h>

enum {
    ORC_GEMM = 0,
    ORC_DISCOUNT = 1,
    ORC_BOOST = 2,
    ORC_SQDIFF = 3,
    ORC_EQCOUNT = 4,
    ORC_THRCOUNT = 5
};

typedef struct {
    const double* p;
    int64_t s0; /* element stride along the statement's first index  */
    int64_t s1; /* element stride along the statement's second index */
} orc_view;

static inline double at(const orc_view* v, int64_t r, int64_t c) { return v->p[r * v->s0 + c * v->s1]; }

static inline double body(int kind, double a, double b, double t, double dis) {
    switch (kind) {
        case ORC_GEMM:
            return a * b;
        case ORC_DISCOUNT: {
            double p = a * b;
            double m = (a * b) > t ? 1.0 : 0.0;
            return p - ((m * a) * b) * dis;
        }
        case ORC_BOOST: {
            double p = a * b;
            double m = (a * b) > t ? 1.0 : 0.0;
            return p + m * ((a * b) - t);
        }
        case ORC_SQDIFF:
            return (a - b) * (a - b);
        case ORC_EQCOUNT:
            return a == b ? 1.0 : 0.0;
        case ORC_THRCOUNT:
            return (a * b) > t ? 1.0 : 0.0;
    }
    return 0.0;
}

/* R(i, j) (+)= sum over k in [k0, k1) of body(A(i,k), B(k,j), T(i,j), D(i,j)),
 * for i in [i0, i1), j in [j0, j1); loops in the reference's declaration
 * order. Returns 0, or -1 for an unknown body. */
int oracle_run(int kind, int accumulate, const orc_view* A, const orc_view* B, const orc_view* T,
               const orc_view* D, double* R, int64_t r_s0, int64_t r_s1, int64_t i0, int64_t i1,
               int64_t j0, int64_t j1, int64_t k0, int64_t k1) {
    if (kind < ORC_GEMM || kind > ORC_THRCOUNT) return -1;
    for (int64_t i = i0; i < i1; ++i) {
        for (int64_t j = j0; j < j1; ++j) {
            double* out = R + i * r_s0 + j * r_s1;
            const double t = T && T->p ? at(T, i, j) : 0.0;
            const double d = D && D->p ? at(D, i, j) : 0.0;
            for (int64_t k = k0; k < k1; ++k) {
                double v = body(kind, at(A, i, k), at(B, k, j), t, d);
                if (accumulate)
                    *out = *out + v;
                else
                    *out = v;
            }
        }
    }
    return 0;
}

/* Scalar evaluation of one body application (SPEC.md:121-123 known answers:
 * discount with A*B=10, thres=5, dis=0.5 -> 5.0; thres=20 -> 10.0). */
double oracle_eval(int kind, double a, double b, double t, double dis) { return body(kind, a, b, t, dis); }
