// naive.cu — the per-element executor: the GPU counterpart of the
// reference's naive interpreter (run_naive, src/naive.cpp:65-117,157-166) and
// of execute_scalar_region (src/kernel_exec.cpp:408-457).
//
// One thread owns one output element R[i][j] and walks k in ascending order,
// evaluating the statement term exactly as the syntax tree does — one
// correctly rounded IEEE operation per tree node, no contraction — then
// `R += v` per term (or `R = v` for assignment statements). It backs the
// "naive" run mode and the --verify check of the command-line front end
// (reference tools/amlt_main.cpp:183-207): an independent, untiled device
// path that the tiled kernels are compared with. It is not a tuning
// candidate and is not tuned for speed beyond coalescing (consecutive
// threads take consecutive j).
#include <cuda_runtime.h>

#include <cstdint>

#include "naive.h"

namespace amltk {
namespace {

template <typename T>
struct Ops {
    static __device__ __forceinline__ T mul(T a, T b) { return a * b; }
    static __device__ __forceinline__ T add(T a, T b) { return a + b; }
    static __device__ __forceinline__ T sub(T a, T b) { return a - b; }
};
template <>
struct Ops<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
};
template <>
struct Ops<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
};

// The statement term for one (i, j, k), in the parse tree's evaluation order
// (presets src/presets.cpp:52-94; left-associative products,
// src/parser.cpp:142-365; comparisons yield 1 / 0, src/naive.cpp:108-112).
template <int BODY, typename T>
__device__ __forceinline__ T term(T a, T b, T t, T dis) {
    using O = Ops<T>;
    if constexpr (BODY == AMLT_BODY_GEMM) {
        return O::mul(a, b);
    } else if constexpr (BODY == AMLT_BODY_DISCOUNT) {
        // A*B - (((A*B > T) * A) * B) * dis
        const T p = O::mul(a, b);
        const T m = p > t ? T(1) : T(0);
        return O::sub(p, O::mul(O::mul(O::mul(m, a), b), dis));
    } else if constexpr (BODY == AMLT_BODY_BOOST) {
        // A*B + (A*B > T) * (A*B - T)
        const T p = O::mul(a, b);
        const T m = p > t ? T(1) : T(0);
        return O::add(p, O::mul(m, O::sub(p, t)));
    } else if constexpr (BODY == AMLT_BODY_SQDIFF) {
        const T d = O::sub(a, b);
        return O::mul(d, d);
    } else if constexpr (BODY == AMLT_BODY_EQCOUNT) {
        return a == b ? T(1) : T(0);
    } else {  // THRCOUNT: (A*B > T)
        return O::mul(a, b) > t ? T(1) : T(0);
    }
}

template <int BODY, typename T>
__global__ void mmlt_naive_kernel(const NaiveParams p) {
    const T* A = static_cast<const T*>(p.A);
    const T* B = static_cast<const T*>(p.B);
    const T* Th = static_cast<const T*>(p.thres);
    const T* Di = static_cast<const T*>(p.dis);
    T* R = static_cast<T*>(p.R);
    const int64_t total = p.M * p.N;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = idx / p.N;
        const int64_t j = idx - i * p.N;
        const T t = Th ? Th[i * p.t_si + j * p.t_sj] : T(p.tconst);
        const T dis = Di ? Di[j * p.d_sj] : T(0);
        T* r = R + i * p.sri + j * p.srj;
        T acc = p.accumulate ? *r : T(0);
        const T* a = A + i * p.sai;
        const T* b = B + j * p.sbj;
        for (int64_t k = 0; k < p.K; ++k) {
            const T v = term<BODY, T>(a[k * p.sak], b[k * p.sbk], t, dis);
            acc = p.accumulate ? Ops<T>::add(acc, v) : v;
        }
        if (p.K > 0 || p.accumulate) *r = acc;
    }
}

template <int BODY, typename T>
cudaError_t launch(const NaiveParams& p, int num_sms, cudaStream_t s) {
    const int64_t total = p.M * p.N;
    if (total == 0) return cudaSuccess;
    const int threads = 256;
    int64_t blocks = (total + threads - 1) / threads;
    blocks = blocks < int64_t(num_sms) * 16 ? blocks : int64_t(num_sms) * 16;
    mmlt_naive_kernel<BODY, T><<<static_cast<unsigned>(blocks), threads, 0, s>>>(p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t by_body(const NaiveParams& p, int body, int num_sms, cudaStream_t s) {
    switch (body) {
        case AMLT_BODY_GEMM: return launch<AMLT_BODY_GEMM, T>(p, num_sms, s);
        case AMLT_BODY_DISCOUNT: return launch<AMLT_BODY_DISCOUNT, T>(p, num_sms, s);
        case AMLT_BODY_BOOST: return launch<AMLT_BODY_BOOST, T>(p, num_sms, s);
        case AMLT_BODY_SQDIFF: return launch<AMLT_BODY_SQDIFF, T>(p, num_sms, s);
        case AMLT_BODY_EQCOUNT: return launch<AMLT_BODY_EQCOUNT, T>(p, num_sms, s);
        case AMLT_BODY_THRCOUNT: return launch<AMLT_BODY_THRCOUNT, T>(p, num_sms, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_naive(const NaiveParams& p, int body, int dtype, int num_sms, cudaStream_t s) {
    if (dtype == AMLT_F64) return by_body<double>(p, body, num_sms, s);
    if (dtype == AMLT_F32) return by_body<float>(p, body, num_sms, s);
    if (body == AMLT_BODY_EQCOUNT) return launch<AMLT_BODY_EQCOUNT, int>(p, num_sms, s);
    if (body == AMLT_BODY_THRCOUNT) return launch<AMLT_BODY_THRCOUNT, int>(p, num_sms, s);
    return cudaErrorInvalidValue;
}

}  // namespace amltk
