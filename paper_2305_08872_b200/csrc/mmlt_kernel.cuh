// mmlt_kernel.cuh — sm_100a CUDA-core kernels for the MMLT loop nest
//
//     R[i][j] (+)= sum_{k in [k0,k1)} body(A[i][k], B[k][j], col_vectors[j])
//
// This is the B200 replacement for the reference's register-blocked kernel
// execute_block / exec_block_t (reference src/kernel_exec.cpp:128-313) and
// its interpreter run_instrs (src/kernel_exec.cpp:63-126), fused per body at
// compile time instead of interpreted per pseudo-instruction.
//
// Structure (one CTA = BM x BN output tile, one thread = TM x TN micro-tile):
//  * A (BM x BK) and B (BK x BN) tiles are staged into shared memory with a
//    STAGES-deep TMA ring (cp.async.bulk.tensor + mbarrier; per-element
//    cp.async for unaligned operands): the reference's packing
//    (src/packing.cpp:5-45) becomes the SMEM copy.
//  * Lanes form an LR x LC grid (LR * LC = 32). LR = 1: every lane of a warp
//    owns the SAME TM rows, so each A read is a 16-byte broadcast and the B
//    reads are lane-interleaved 16-byte vectors (32 distinct per load: four
//    wavefronts). LR > 1: the LR lanes of a column group share its B vectors
//    (one wavefront per load) and read LR distinct A rows, conflict-free
//    through the TMA 128-byte swizzle of the A tile. Shared-memory traffic
//    per product drops about threefold for the 8 x 4 f64 micro-tile, which is
//    what bounds the three-plane theta-form discount.
//  * The per-j vectors (thres[j], dis[j]) are loaded once into registers.
//  * The body is fused into the accumulate chain on CUDA cores (tensor cores
//    cannot evaluate a per-product predicate); see the Body structs below for
//    the exact per-iteration instruction mix each one compiles to.
//  * K tail tiles run a guarded loop (operands past k1 are never applied, so
//    bodies like A == B do not count zero padding).
//  * Split-K (TileParams.kc < K) writes per-segment partials to a workspace
//    reduced in segment order by mmlt_splitk_reduce: deterministic.
#pragma once

#ifndef __CUDACC_RTC__
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#else
// Compiled at run time by NVRTC for generated bodies (csrc/jit.cu): no host
// headers, so the few types the kernels use are declared here.
typedef long long int64_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef unsigned long long uintptr_t;
struct alignas(64) CUtensorMap_st {
    unsigned long long opaque[16];
};
typedef CUtensorMap_st CUtensorMap;
#endif

// Aux leaves of a generated (generic) body: at most this many arrays.
#define AMLT_KP_MAX_AUX 8

namespace amltk {

// --------------------------------------------------------------------------
// Launch parameters (plain data, passed by value)

struct KParams {
    const void* A;  // A(i, k) at A[i * lda + k], already offset to (i0, k0)
    const void* B;  // B(k, j) at B[k * ldb + j], already offset to (k0, j0)
    void* R;        // R(i, j) at R[i * ldr + j], already offset to (i0, j0)
    const void* thres;  // T(j) at thres[j * t_sj] (t_sj == 0: broadcast scalar)
    const void* dis;    // dis(j) at dis[j * d_sj]
    void* work;         // split-K workspace: [splits][M][N] of T
    int64_t lda, ldb, ldr;
    int64_t t_sj, d_sj;
    int64_t t_si;      // threshold row stride (T indexed by i or by (i, j)); 0 otherwise
    int64_t M, N, K;   // extents of the bounds rectangle
    int64_t kslice;    // K depth per split (== K when splits == 1)
    int32_t splits;
    int32_t tiles_m, tiles_n;
    int32_t group_m;   // row tiles per raster group (L2 reuse of B panels)
    int32_t r_vec_ok;  // R base 16B aligned and ldr a multiple of the vector width
    double tconst;     // threshold when thres == nullptr
    // Generated bodies (AMLT_BODY_GENERIC): aux leaf q of output (i, j) is
    // gaux[q][i * gaux_si[q] + j * gaux_sj[q]], offset to (i0, j0).
    const void* gaux[AMLT_KP_MAX_AUX];
    int64_t gaux_si[AMLT_KP_MAX_AUX];
    int64_t gaux_sj[AMLT_KP_MAX_AUX];
    // Guarded variants (theta-form discount and its fallback): operand range
    // statistics the kernels read to decide which of the two runs.
    const int* guard;
    // R starts at zero: the epilogue writes 0 + value and never reads R (a
    // result written straight to mapped host memory needs no memset there)
    int32_t r_zero;
    // Variants with a prepared copy of B (VariantDesc::prep_panels): this
    // launch's k rows start at row plane_k0 of a preparation plane_kdim rows
    // deep (0: the preparation is exactly this launch's K range).
    int64_t plane_k0;
    int64_t plane_kdim;
};

// --------------------------------------------------------------------------
// cp.async helpers (LDGSTS). src_bytes < size zero-fills the remainder.

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
                 "r"(src_bytes));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_elem(void* smem, const void* gmem, int src_bytes) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem),
                 "n"(BYTES), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// 16-byte vector of T
template <typename T>
struct V16;
template <>
struct V16<double> {
    using type = double2;
    static constexpr int n = 2;
    __device__ static __forceinline__ double get(const double2& v, int e) { return e == 0 ? v.x : v.y; }
};
template <>
struct V16<float> {
    using type = float4;
    static constexpr int n = 4;
    __device__ static __forceinline__ float get(const float4& v, int e) {
        return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
    }
};
template <>
struct V16<int> {
    using type = int4;
    static constexpr int n = 4;
    __device__ static __forceinline__ int get(const int4& v, int e) {
        return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
    }
};

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
__device__ __forceinline__ float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }

template <typename T>
__device__ __forceinline__ T ldg_elem(const void* base, int64_t idx) {
    return __ldg(static_cast<const T*>(base) + idx);
}

template <typename T>
struct IsF32 {
    static constexpr bool value = false;
};
template <>
struct IsF32<float> {
    static constexpr bool value = true;
};

// Counting bodies: acc += (x CMP y), as SETP + predicated add — two issue
// slots (nvcc's own lowering of `acc += cond ? 1 : 0` is a speculative add
// plus a predicated move, three).
constexpr int CMP_EQ = 0;
constexpr int CMP_GT = 1;
template <int CMP>
__device__ __forceinline__ void inc_if(int& acc, int x, int y) {
    if constexpr (CMP == CMP_EQ)
        asm("{\n .reg .pred p;\n setp.eq.s32 p, %1, %2;\n @p add.s32 %0, %0, 1;\n}\n"
            : "+r"(acc) : "r"(x), "r"(y));
    else
        asm("{\n .reg .pred p;\n setp.gt.s32 p, %1, %2;\n @p add.s32 %0, %0, 1;\n}\n"
            : "+r"(acc) : "r"(x), "r"(y));
}
template <int CMP>
__device__ __forceinline__ void inc_if(int& acc, float x, float y) {
    if constexpr (CMP == CMP_EQ)
        asm("{\n .reg .pred p;\n setp.eq.f32 p, %1, %2;\n @p add.s32 %0, %0, 1;\n}\n"
            : "+r"(acc) : "f"(x), "f"(y));
    else
        asm("{\n .reg .pred p;\n setp.gt.f32 p, %1, %2;\n @p add.s32 %0, %0, 1;\n}\n"
            : "+r"(acc) : "f"(x), "f"(y));
}
template <int CMP>
__device__ __forceinline__ void inc_if(int& acc, double x, double y) {
    if constexpr (CMP == CMP_EQ)
        asm("{\n .reg .pred p;\n setp.eq.f64 p, %1, %2;\n @p add.s32 %0, %0, 1;\n}\n"
            : "+r"(acc) : "d"(x), "d"(y));
    else
        asm("{\n .reg .pred p;\n setp.gt.f64 p, %1, %2;\n @p add.s32 %0, %0, 1;\n}\n"
            : "+r"(acc) : "d"(x), "d"(y));
}

// --------------------------------------------------------------------------
// Bodies. Each gives the per-(i,j,k) update on the accumulators of one
// output element, the per-column state it needs, and the final value added
// to R. The reference statement, its compiled pseudo-program (schedule.cpp
// output) and the B200 instruction mix are listed per body.

// GEMM — `R[i][j] += A[i][k]*B[k][j]` (preset matmul; ref program
// `mul REG0 A B; add R R REG0`, fused FMA path kernel_exec.cpp:161-178).
// B200: 1 FFMA/DFMA per iteration.
template <typename T>
struct BodyGemm {
    using Acc = T;
    static constexpr int NACC = 1;
    // One accumulator level: GEMM's tolerance is normwise (|d| <= tol * sum |a b|,
    // SURVEY §7), where sequential fp32 accumulation at K = 8192 stays ~100x
    // inside 1e-5; the registers go to a larger micro-tile instead.
    static constexpr bool TWO_LEVEL = false;
    struct Col {};
    __device__ static Col col(const KParams&, int64_t) { return {}; }
    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col&) {
        acc[0] = fma_rn(a, b, acc[0]);
    }
    // fp32: two columns per FFMA2 (half the issue slots, the same FMA-pipe work)
    static constexpr bool PAIRED = IsF32<T>::value;
    __device__ static __forceinline__ void step2(Acc* acc0, Acc* acc1, T a, T b0, T b1, const Col&, const Col&) {
        asm("{\n .reg .b64 x, y, s;\n"
            " mov.b64 x, {%2, %2};\n mov.b64 y, {%3, %4};\n mov.b64 s, {%0, %1};\n"
            " fma.rn.f32x2 s, x, y, s;\n mov.b64 {%0, %1}, s;\n}\n"
            : "+f"(acc0[0]), "+f"(acc1[0])
            : "f"(a), "f"(b0), "f"(b1));
    }
    __device__ static __forceinline__ T finish(const Acc* acc, const Col&, int64_t) { return acc[0]; }
};

// DISCOUNT — preset q1: `R += A*B - (A*B > thres[j])*A*B*dis[j]`
// (presets.cpp:66-67; ref program `mul; gtcmp; mul; masksub; add`).
// Per product p = A*B (rounded exactly as the reference rounds it, so the
// mask never flips): acc += p * (p > t ? 1 - dis : 1).
// B200: DMUL + DSETP + DFMA on the FP64 pipe, 2 FSEL on the ALU pipe.
template <typename T>
struct BodyDiscount {
    using Acc = T;
    static constexpr int NACC = 1;
    static constexpr bool TWO_LEVEL = sizeof(T) == 4;
    struct Col {
        T t, c1;
    };
    __device__ static Col col(const KParams& p, int64_t j) {
        Col c;
        c.t = p.thres ? ldg_elem<T>(p.thres, j * p.t_sj) : static_cast<T>(p.tconst);
        c.c1 = T(1) - ldg_elem<T>(p.dis, j * p.d_sj);
        return c;
    }
    static constexpr bool USES_T = true;
    __device__ static __forceinline__ Col with_t(Col c, T t) {
        c.t = t;
        return c;
    }
    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col& c) {
        T pr = mul_rn(a, b);
        T f = pr > c.t ? c.c1 : T(1);
        acc[0] = fma_rn(pr, f, acc[0]);
    }
    __device__ static __forceinline__ T finish(const Acc* acc, const Col&, int64_t) { return acc[0]; }
};

// BOOST — preset q2: `R += A*B + (A*B > thres[j])*(A*B - thres[j])`
// (presets.cpp:68-69; ref program `mul; gtcmp; sub; maskadd; add`).
// The mask term is relu(p - t) = ((p - t) + |p - t|) / 2, continuous at the
// threshold. Summed over the K segment:
//   sum relu(u_k) = (sum_k (a b - t) + sum_k |u_k|) / 2
//                 = (acc0 - kcount*t + acc1) / 2
// with acc0 = sum a*b (FMA) and acc1 = sum |fma(a, b, -t)|; |.| is a free
// operand modifier. B200: 3 FP pipe ops per iteration (FMA, FMA, ADD), no ALU
// selects at all.
template <typename T>
struct BodyBoost {
    using Acc = T;
    static constexpr int NACC = 2;
    static constexpr bool TWO_LEVEL = sizeof(T) == 4;
    struct Col {
        T t, nt;
    };
    __device__ static Col col(const KParams& p, int64_t j) {
        Col c;
        c.t = p.thres ? ldg_elem<T>(p.thres, j * p.t_sj) : static_cast<T>(p.tconst);
        c.nt = -c.t;
        return c;
    }
    static constexpr bool USES_T = true;
    __device__ static __forceinline__ Col with_t(Col c, T t) {
        c.t = t;
        c.nt = -t;
        return c;
    }
    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col& c) {
        acc[0] = fma_rn(a, b, acc[0]);
        T u = fma_rn(a, b, c.nt);
        acc[1] = add_rn(acc[1], fabs(u));
    }
    __device__ static __forceinline__ T finish(const Acc* acc, const Col& c, int64_t kcount) {
        T s = acc[0] - static_cast<T>(kcount) * c.t;  // sum of (a*b - t)
        return acc[0] + T(0.5) * (s + acc[1]);
    }
    // (A two-column fp32 form, FFMA2 + FFMA2 + FADD2, needs |u| as a sign
    // mask: two LOP3 per pair on the ALU. Measured 17.8 against 19.9 TFLOP/s
    // at 4096^3, so boost keeps the one-column step with its free |.|.)
};

// SQDIFF — `R += (A - B)*(A - B)`: FADD + FFMA per iteration; in fp32 two
// columns at a time as FADD2 + FFMA2 (sm_100's two-wide fp32 instructions:
// the same FMA-pipe work in half the issue slots).
template <typename T>
struct BodySqdiff {
    using Acc = T;
    static constexpr int NACC = 1;
    static constexpr bool TWO_LEVEL = sizeof(T) == 4;
    static constexpr bool PAIRED = IsF32<T>::value;
    struct Col {};
    __device__ static Col col(const KParams&, int64_t) { return {}; }
    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col&) {
        T d = a - b;
        acc[0] = fma_rn(d, d, acc[0]);
    }
    // columns c and c+1 of one row: acc0 / acc1
    __device__ static __forceinline__ void step2(Acc* acc0, Acc* acc1, T a, T b0, T b1, const Col&, const Col&) {
        asm("{\n .reg .b64 x, y, s, d;\n"
            " mov.b64 x, {%2, %2};\n mov.b64 y, {%3, %4};\n mov.b64 s, {%0, %1};\n"
            " sub.rn.f32x2 d, x, y;\n fma.rn.f32x2 s, d, d, s;\n mov.b64 {%0, %1}, s;\n}\n"
            : "+f"(acc0[0]), "+f"(acc1[0])
            : "f"(a), "f"(b0), "f"(b1));
    }
    __device__ static __forceinline__ T finish(const Acc* acc, const Col&, int64_t) { return acc[0]; }
};

// EQCOUNT — `R += A == B` (ref program `eqcmp; maskadd $0 $1; add`).
// Integer accumulator: ISETP + predicated add. Float/double inputs count in
// int32 too (the count is exact; K < 2^31) and convert at the end.
template <typename T>
struct BodyEqcount {
    using Acc = int;
    static constexpr int NACC = 1;
    static constexpr bool TWO_LEVEL = false;
    struct Col {};
    __device__ static Col col(const KParams&, int64_t) { return {}; }
    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col&) {
        inc_if<CMP_EQ>(acc[0], a, b);
    }
    __device__ static __forceinline__ T finish(const Acc* acc, const Col&, int64_t) {
        return static_cast<T>(acc[0]);
    }
};

// THRCOUNT — preset q3: `R += (A*B > 100)` (presets.cpp:70-71).
template <typename T>
struct BodyThrcount {
    using Acc = int;
    static constexpr int NACC = 1;
    static constexpr bool TWO_LEVEL = false;
    struct Col {
        T t;
    };
    __device__ static Col col(const KParams& p, int64_t j) {
        Col c;
        c.t = p.thres ? ldg_elem<T>(p.thres, j * p.t_sj) : static_cast<T>(p.tconst);
        return c;
    }
    static constexpr bool USES_T = true;
    __device__ static __forceinline__ Col with_t(Col c, T t) {
        c.t = t;
        return c;
    }
    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col& c) {
        inc_if<CMP_GT>(acc[0], mul_rn(a, b), c.t);
    }
    __device__ static __forceinline__ T finish(const Acc* acc, const Col&, int64_t) {
        return static_cast<T>(acc[0]);
    }
};
template <>
__device__ __forceinline__ void BodyThrcount<int>::step(int* acc, int a, int b, const Col& c) {
    inc_if<CMP_GT>(acc[0], a * b, c.t);
}

// Bodies with a threshold operand T (discount, boost, thrcount).
template <class Body, class = void>
struct UsesThreshold {
    static constexpr bool value = false;
};
template <class Body>
struct UsesThreshold<Body, decltype(void(Body::USES_T))> {
    static constexpr bool value = Body::USES_T;
};

// Generated bodies with aux leaves indexed by i or (i, j) complete their
// column state per output element (Body::at).
template <class Body, class = void>
struct HasAt {
    static constexpr bool value = false;
};
template <class Body>
struct HasAt<Body, decltype(void(Body::HAS_AT))> {
    static constexpr bool value = Body::HAS_AT;
};

// Two-level bodies may fold the per-BK-tile partial into the running
// accumulator their own way (FOLD: Body::fold(acc, part)); the default adds.
template <class Body, class = void>
struct BodyFold {
    template <typename Acc>
    __device__ static __forceinline__ void go(Acc& acc, const Acc& part) {
        acc += part;
    }
};
template <class Body>
struct BodyFold<Body, decltype(void(Body::FOLD))> {
    template <typename Acc>
    __device__ static __forceinline__ void go(Acc& acc, const Acc& part) {
        Body::fold(acc, part);
    }
};

// Bodies whose B operand is a prepared multi-plane array (BPLANES planes of
// K x N, one TMA box per stage covers all planes).
template <class Body, class = void>
struct BodyPlanes {
    static constexpr int n = 1;
};
template <class Body>
struct BodyPlanes<Body, decltype(void(Body::BPLANES))> {
    static constexpr int n = Body::BPLANES;
};

// Bodies with a two-column step (Body::step2, e.g. fp32 FFMA2 forms).
template <class Body, class = void>
struct Paired {
    static constexpr bool value = false;
};
template <class Body>
struct Paired<Body, decltype(void(Body::PAIRED))> {
    static constexpr bool value = Body::PAIRED;
};

// Bodies whose inner step runs row-outer (the row's a is the shared operand
// of consecutive instructions) instead of the default column-outer order.
template <class Body, class = void>
struct RowOuter {
    static constexpr bool value = false;
};
template <class Body>
struct RowOuter<Body, decltype(void(Body::ROW_OUTER))> {
    static constexpr bool value = Body::ROW_OUTER;
};

// Bodies that run only when Body::guard(p) holds (checked once per CTA).
template <class Body, class = void>
struct BodyGuard {
    __device__ static __forceinline__ bool run(const KParams&) { return true; }
};
template <class Body>
struct BodyGuard<Body, decltype(void(Body::GUARDED))> {
    __device__ static __forceinline__ bool run(const KParams& p) { return Body::guard(p); }
};

// Column state with the threshold of output (i, j) when T is indexed by i or
// by (i, j): T(i, j) = thres[i * t_si + j * t_sj] (TCLS == 1 kernels).
template <class Body, typename T>
__device__ __forceinline__ typename Body::Col col_at(const typename Body::Col& c, const KParams& p,
                                                     int64_t i, int64_t j) {
    if constexpr (HasAt<Body>::value)
        return Body::at(c, p, i, j);
    else if constexpr (UsesThreshold<Body>::value)
        return Body::with_t(c, ldg_elem<T>(p.thres, i * p.t_si + j * p.t_sj));
    else
        return c;
}

// --------------------------------------------------------------------------
// TMA + mbarrier helpers (sm_90+ PTX; on sm_100a the copies are UTMALDG)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// One body step with the B planes of the current (k, j): plane 0 is b itself
// for single-plane bodies.
template <class Body, int NPL>
struct PlaneStep {
    template <typename Acc, typename T, typename Col>
    __device__ static __forceinline__ void go(Acc* acc, T a, T b0, T, T, const Col& col) {
        Body::step(acc, a, b0, col);
    }
};
template <class Body>
struct PlaneStep<Body, 3> {
    template <typename Acc, typename T, typename Col>
    __device__ static __forceinline__ void go(Acc* acc, T a, T b0, T b1, T b2, const Col&) {
        Body::step3(acc, a, b0, b1, b2);
    }
};

__device__ __forceinline__ void tma_load_planes(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                                uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(0), "r"(smem_u32(bar))
        : "memory");
}

// --------------------------------------------------------------------------
// The tiled kernel
//
// LOAD selects the staging path:
//   LOAD_TMA   one thread issues two cp.async.bulk.tensor copies per stage (A
//              box BK x BM, B box BN x BK) that complete on the stage's
//              mbarrier; out-of-range rows/columns arrive zero-filled. No
//              per-thread address arithmetic in the main loop.
//   LOAD_ELEM  per-element cp.async (4/8-byte LDGSTS) for operands whose base
//              or leading dimension is not 16-byte aligned.

constexpr int LOAD_ELEM = 0;
constexpr int LOAD_TMA = 1;
// flag: per-output threshold state (T indexed by i or by (i, j))
constexpr int LOAD_TOUT = 2;
// lane grid: bits 2-3 hold log2(LR), LR lanes along rows (see the header)
constexpr int LOAD_LR2 = 1 << 2;
constexpr int LOAD_LR4 = 2 << 2;
constexpr int LOAD_LR8 = 3 << 2;
__host__ __device__ constexpr int load_lr(int load) { return 1 << ((load >> 2) & 3); }

template <class Body, typename T, int TM, int TN, int WR, int WC, int BK, int STAGES, int LOAD,
          int MINB>
struct MmltTile {
    static constexpr int VN = V16<T>::n;
    static constexpr int THREADS = 32 * WR * WC;
    static constexpr int LR = load_lr(LOAD);  // lanes along rows
    static constexpr int LC = 32 / LR;        // lanes along columns
    static constexpr bool SWZ = LR > 1;       // A tile in the TMA 128-byte swizzle
    static constexpr int BM = TM * LR * WR;
    static constexpr int BN = LC * TN * WC;
    static constexpr int SMEM_A = BM * BK;  // elements per stage
    static constexpr int NPL = BodyPlanes<Body>::n;
    static constexpr int SMEM_B = BK * BN * NPL;
    static constexpr int BAR_BYTES = 16 * STAGES;  // full + empty mbarriers (within the +128)
    // + 1024: the swizzled A stages start on a 1024-byte boundary
    static constexpr int SMEM_BYTES = STAGES * (SMEM_A + SMEM_B) * (int)sizeof(T) + 128 + (SWZ ? 1024 : 0);
    static_assert(TN % VN == 0, "TN must be a multiple of the 16B vector width");
    static_assert(BK % VN == 0, "BK must be a multiple of the 16B vector width");
    static_assert(STAGES >= 2, "need at least double buffering");
    static_assert((SMEM_A * sizeof(T)) % 128 == 0, "TMA stage buffers must stay 128B aligned");
    static_assert(BN <= 256 && BM <= 256 && BK <= 256, "TMA box dims are at most 256");
    static_assert(NPL == 1 || ((LOAD & LOAD_TMA) != 0 && (LOAD & LOAD_TOUT) == 0),
                  "multi-plane B is TMA-staged with per-column state only");
    static_assert(!SWZ || ((LOAD & LOAD_TMA) != 0 && BK * (int)sizeof(T) == 128 && TM * LR % 8 == 0),
                  "the 2-D lane grid reads a TMA-swizzled A tile of 128-byte rows");
    static_assert(!SWZ || LC * VN * (int)sizeof(T) <= 128, "a column group's B load must stay one wavefront");
    // element offset of A(row, k) inside a stage (the TMA 128B swizzle XORs
    // the 16-byte chunk index with row % 8)
    __device__ static __forceinline__ int a_off(int row, int k) {
        if constexpr (SWZ)
            return row * BK + ((((k / VN) ^ (row & 7)) * VN) | (k % VN));
        else
            return row * BK + k;
    }
};

template <class Body, typename T, int TM, int TN, int WR, int WC, int BK, int STAGES, int LOAD,
          int MINB>
__global__ void __launch_bounds__(32 * WR * WC, MINB)
    mmlt_tile_kernel(const __grid_constant__ KParams p, const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB) {
    using Cfg = MmltTile<Body, T, TM, TN, WR, WC, BK, STAGES, LOAD, MINB>;
    constexpr bool TOUT = (LOAD & LOAD_TOUT) != 0;
    constexpr int VN = Cfg::VN;
    constexpr int THREADS = Cfg::THREADS;
    constexpr int BM = Cfg::BM;
    constexpr int BN = Cfg::BN;
    using Vec = typename V16<T>::type;
    using Acc = typename Body::Acc;
    constexpr int NACC = Body::NACC;
    constexpr int NPL = Cfg::NPL;
    if (!BodyGuard<Body>::run(p)) return;  // CTA-uniform: before any barrier setup

    extern __shared__ __align__(128) unsigned char smem_raw_[];
    unsigned char* smem_raw = smem_raw_;
    if constexpr (Cfg::SWZ)
        smem_raw += (1024 - (smem_u32(smem_raw_) & 1023)) & 1023;
    T* As = reinterpret_cast<T*>(smem_raw);
    T* Bs = As + STAGES * Cfg::SMEM_A;
    uint64_t* full = reinterpret_cast<uint64_t*>(Bs + STAGES * Cfg::SMEM_B);
    // per-stage count of warps done reading it: the last one refills it
    unsigned int* done = reinterpret_cast<unsigned int*>(full + STAGES);

    // ---- tile coordinates: grouped raster (group_m row-tiles per group, about
    // 512 rows) so the B column panels of concurrently resident CTAs are
    // shared through L2 while the group's A rows also stay resident.
    const int G = p.group_m;
    const int bid = blockIdx.x;
    const int per_group = G * p.tiles_n;
    const int group = bid / per_group;
    const int first_m = group * G;
    const int gsize = min(p.tiles_m - first_m, G);
    const int in_group = bid - group * per_group;
    const int tile_m = first_m + in_group % gsize;
    const int tile_n = in_group / gsize;
    const int64_t m0 = static_cast<int64_t>(tile_m) * BM;
    const int64_t n0 = static_cast<int64_t>(tile_n) * BN;

    const int split = blockIdx.y;
    const int64_t kbeg = static_cast<int64_t>(split) * p.kslice;
    const int64_t kspan = min(p.kslice, p.K - kbeg);

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int wr = warp / WC;
    const int wc = warp - wr * WC;
    constexpr int LR = Cfg::LR, LC = Cfg::LC;
    const int lg = LR > 1 ? lane % LR : 0;  // row slot in the lane grid
    const int lh = LR > 1 ? lane / LR : lane;  // column group
    // this thread's rows: row0 + r * LR (interleaved, so the LR lanes of a
    // column group hit distinct swizzle phases); columns: col0 + q * LC * VN + e
    const int row0 = wr * TM * LR + lg;
    const int col0 = wc * LC * TN + lh * VN;

    const T* __restrict__ Ag = static_cast<const T*>(p.A);
    const T* __restrict__ Bg = static_cast<const T*>(p.B);
    const int nkt = static_cast<int>((kspan + BK - 1) / BK);

    // ---- stage loaders
    constexpr uint32_t STAGE_TX = (Cfg::SMEM_A + Cfg::SMEM_B) * sizeof(T);
    auto tma_stage = [&](int stage, int kt) {  // called by one thread
        mbar_expect_tx(&full[stage], STAGE_TX);
        const int32_t k = static_cast<int32_t>(kbeg + static_cast<int64_t>(kt) * BK);
        tma_load_2d(As + stage * Cfg::SMEM_A, &tmA, k, static_cast<int32_t>(m0), &full[stage]);
        if constexpr (NPL == 1)
            tma_load_2d(Bs + stage * Cfg::SMEM_B, &tmB, static_cast<int32_t>(n0), k, &full[stage]);
        else
            tma_load_planes(Bs + stage * Cfg::SMEM_B, &tmB, static_cast<int32_t>(n0), k, &full[stage]);
    };
    auto elem_stage = [&](int stage, int kt) {  // called by all threads
        T* as = As + stage * Cfg::SMEM_A;
        T* bs = Bs + stage * Cfg::SMEM_B;
        const int64_t k0 = kbeg + static_cast<int64_t>(kt) * BK;
        const int64_t kend = kbeg + kspan;
        for (int c = tid; c < BM * BK; c += THREADS) {
            const int row = c / BK;
            const int kc = c - row * BK;
            const int64_t gi = m0 + row;
            const int64_t gk = k0 + kc;
            const bool ok = gi < p.M && gk < kend;
            cp_async_elem<sizeof(T)>(as + row * BK + kc, ok ? Ag + gi * p.lda + gk : Ag,
                                     ok ? (int)sizeof(T) : 0);
        }
        for (int c = tid; c < BK * BN; c += THREADS) {
            const int kr = c / BN;
            const int cc = c - kr * BN;
            const int64_t gk = k0 + kr;
            const int64_t gj = n0 + cc;
            const bool ok = gk < kend && gj < p.N;
            cp_async_elem<sizeof(T)>(bs + kr * BN + cc, ok ? Bg + gk * p.ldb + gj : Bg,
                                     ok ? (int)sizeof(T) : 0);
        }
    };

    if constexpr ((LOAD & LOAD_TMA) != 0) {
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < STAGES; ++s) {
                mbar_init(&full[s], 1);
                done[s] = 0;
            }
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
        }
        __syncthreads();
        if (tid == 0) {
#pragma unroll
            for (int s = 0; s < STAGES; ++s)
                if (s < nkt) tma_stage(s, s);
        }
    } else {
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < nkt) elem_stage(s, s);
            cp_async_commit();
        }
    }

    // ---- per-thread columns: local col of element (q, e) is col0 + q*LC*VN + e
    typename Body::Col colst[TN];
#pragma unroll
    for (int q = 0; q < TN / VN; ++q)
#pragma unroll
        for (int e = 0; e < VN; ++e) {
            const int64_t gj = n0 + col0 + q * LC * VN + e;
            colst[q * VN + e] = Body::col(p, gj < p.N ? gj : 0);
        }
    // Thresholds indexed by i or (i, j) (LOAD_TOUT variants): one state per
    // output element, loaded once.
    typename Body::Col colrc[TOUT ? TM : 1][TOUT ? TN : 1];
    if constexpr (TOUT) {
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
            for (int q = 0; q < TN / VN; ++q)
#pragma unroll
                for (int e = 0; e < VN; ++e) {
                    const int64_t gi = m0 + row0 + r * LR;
                    const int64_t gj = n0 + col0 + q * LC * VN + e;
                    colrc[r][q * VN + e] = col_at<Body, T>(colst[q * VN + e], p, gi < p.M ? gi : 0,
                                                           gj < p.N ? gj : 0);
                }
    }
#define STEP_PLANES(accv, a_, c_, col_) \
    PlaneStep<Body, NPL>::go(accv, a_, b[c_], bx[0][c_], bx[NPL > 2 ? 1 : 0][c_], col_)
#define COL(r, c) (TOUT ? colrc[TOUT ? (r) : 0][TOUT ? (c) : 0] : colst[c])
#define STEP(accv, a_, c_, col_) STEP_PLANES(accv, a_, c_, col_)

    Acc acc[TM][TN][NACC];
    Acc part[Body::TWO_LEVEL ? TM : 1][Body::TWO_LEVEL ? TN : 1][NACC];
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c)
#pragma unroll
            for (int n = 0; n < NACC; ++n) acc[r][c][n] = Acc(0);
    if constexpr (Body::TWO_LEVEL) {
#pragma unroll
        for (int r = 0; r < TM; ++r)
#pragma unroll
            for (int c = 0; c < TN; ++c)
#pragma unroll
                for (int n = 0; n < NACC; ++n) part[r][c][n] = Acc(0);
    }

    for (int kt = 0; kt < nkt; ++kt) {
        const int stage = kt % STAGES;
        if constexpr ((LOAD & LOAD_TMA) != 0) {
            mbar_wait(&full[stage], static_cast<uint32_t>((kt / STAGES) & 1));
        } else {
            cp_async_wait<STAGES - 2>();
            __syncthreads();
            const int nxt = kt + STAGES - 1;
            if (nxt < nkt) elem_stage(nxt % STAGES, nxt);
            cp_async_commit();
        }
        const T* as = As + stage * Cfg::SMEM_A;
        const T* bs = Bs + stage * Cfg::SMEM_B + col0;
        const int kcount =
            static_cast<int>(min(static_cast<int64_t>(BK), kspan - static_cast<int64_t>(kt) * BK));

        if (kcount == BK) {
#pragma unroll
            for (int kk = 0; kk < BK; kk += VN) {
                Vec av[TM];
#pragma unroll
                for (int r = 0; r < TM; ++r) av[r] = *reinterpret_cast<const Vec*>(as + Cfg::a_off(row0 + r * LR, kk));
#pragma unroll
                for (int v = 0; v < VN; ++v) {
                    T b[TN];
                    T bx[NPL > 1 ? NPL - 1 : 1][TN] = {};
#pragma unroll
                    for (int q = 0; q < TN / VN; ++q) {
                        Vec bv = *reinterpret_cast<const Vec*>(bs + (kk + v) * BN + q * LC * VN);
#pragma unroll
                        for (int e = 0; e < VN; ++e) b[q * VN + e] = V16<T>::get(bv, e);
#pragma unroll
                        for (int pl = 1; pl < NPL; ++pl) {
                            Vec xv = *reinterpret_cast<const Vec*>(bs + pl * BK * BN + (kk + v) * BN + q * LC * VN);
#pragma unroll
                            for (int e = 0; e < VN; ++e) bx[pl - 1][q * VN + e] = V16<T>::get(xv, e);
                        }
                    }
                    if constexpr (RowOuter<Body>::value) {
#pragma unroll
                        for (int r = 0; r < TM; ++r) {
                            const T a = V16<T>::get(av[r], v);
#pragma unroll
                            for (int c = 0; c < TN; ++c) {
                                if constexpr (Body::TWO_LEVEL)
                                    STEP(part[r][c], a, c, COL(r, c));
                                else
                                    STEP(acc[r][c], a, c, COL(r, c));
                            }
                        }
                    } else if constexpr (Paired<Body>::value && NPL == 1 && TN % 2 == 0) {
#pragma unroll
                        for (int c = 0; c < TN; c += 2) {
#pragma unroll
                            for (int r = 0; r < TM; ++r) {
                                const T a = V16<T>::get(av[r], v);
                                if constexpr (Body::TWO_LEVEL)
                                    Body::step2(part[r][c], part[r][c + 1], a, b[c], b[c + 1], COL(r, c), COL(r, c + 1));
                                else
                                    Body::step2(acc[r][c], acc[r][c + 1], a, b[c], b[c + 1], COL(r, c), COL(r, c + 1));
                            }
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < TN; ++c) {
#pragma unroll
                            for (int r = 0; r < TM; ++r) {
                                const T a = V16<T>::get(av[r], v);
                                if constexpr (Body::TWO_LEVEL)
                                    STEP(part[r][c], a, c, COL(r, c));
                                else
                                    STEP(acc[r][c], a, c, COL(r, c));
                            }
                        }
                    }
                }
            }
        } else {
            for (int k = 0; k < kcount; ++k) {
                T b[TN];
                T bx[NPL > 1 ? NPL - 1 : 1][TN] = {};
#pragma unroll
                for (int q = 0; q < TN / VN; ++q) {
                    Vec bv = *reinterpret_cast<const Vec*>(bs + k * BN + q * LC * VN);
#pragma unroll
                    for (int e = 0; e < VN; ++e) b[q * VN + e] = V16<T>::get(bv, e);
#pragma unroll
                    for (int pl = 1; pl < NPL; ++pl) {
                        Vec xv = *reinterpret_cast<const Vec*>(bs + pl * BK * BN + k * BN + q * LC * VN);
#pragma unroll
                        for (int e = 0; e < VN; ++e) bx[pl - 1][q * VN + e] = V16<T>::get(xv, e);
                    }
                }
#pragma unroll
                for (int r = 0; r < TM; ++r) {
                    const T a = as[Cfg::a_off(row0 + r * LR, k)];
#pragma unroll
                    for (int c = 0; c < TN; ++c) {
                        if constexpr (Body::TWO_LEVEL)
                            STEP(part[r][c], a, c, COL(r, c));
                        else
                            STEP(acc[r][c], a, c, COL(r, c));
                    }
                }
            }
        }
        if constexpr (Body::TWO_LEVEL) {
#pragma unroll
            for (int r = 0; r < TM; ++r)
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int n = 0; n < NACC; ++n) {
                        BodyFold<Body>::go(acc[r][c][n], part[r][c][n]);
                        part[r][c][n] = Acc(0);
                    }
        }
        if constexpr ((LOAD & LOAD_TMA) != 0) {
            // this warp is done reading the stage; the LAST warp to finish it
            // refills it with tile kt+STAGES (no CTA-wide barrier and nobody
            // waits: warps drift across the ready stages)
            __syncwarp();
            if (lane == 0) {
                asm volatile("fence.acq_rel.cta;\n" ::: "memory");  // our reads before the count
                if (atomicAdd(&done[stage], 1u) == THREADS / 32 - 1) {
                    done[stage] = 0;
                    // every warp's reads before the async-proxy (TMA) overwrite
                    asm volatile("fence.acq_rel.cta;\n" ::: "memory");
                    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
                    if (kt + STAGES < nkt) tma_stage(stage, kt + STAGES);
                }
            }
        }
    }
    if constexpr ((LOAD & LOAD_TMA) == 0) cp_async_wait<0>();

    // ---- epilogue: R (+)= value, or the split-K workspace
    T* Rg = static_cast<T*>(p.R);
    T* Wg = static_cast<T*>(p.work);
#pragma unroll
    for (int r = 0; r < TM; ++r) {
        const int64_t gi = m0 + row0 + r * LR;
        if (gi >= p.M) continue;
#pragma unroll
        for (int q = 0; q < TN / VN; ++q) {
            const int64_t gj0 = n0 + col0 + q * LC * VN;
            T val[VN];
#pragma unroll
            for (int e = 0; e < VN; ++e) val[e] = Body::finish(acc[r][q * VN + e], COL(r, q * VN + e), kspan);
            if (p.splits > 1) {
                T* dst = Wg + (static_cast<int64_t>(split) * p.M + gi) * p.N + gj0;
#pragma unroll
                for (int e = 0; e < VN; ++e)
                    if (gj0 + e < p.N) dst[e] = val[e];
            } else {
                T* dst = Rg + gi * p.ldr + gj0;
                if (p.r_vec_ok && gj0 + VN <= p.N) {
                    Vec o;
                    if (p.r_zero) {
                        T* op = reinterpret_cast<T*>(&o);
#pragma unroll
                        for (int e = 0; e < VN; ++e) op[e] = T(0);
                    } else {
                        o = *reinterpret_cast<const Vec*>(dst);
                    }
                    T* op = reinterpret_cast<T*>(&o);
#pragma unroll
                    for (int e = 0; e < VN; ++e) op[e] = op[e] + val[e];
                    *reinterpret_cast<Vec*>(dst) = o;
                } else {
#pragma unroll
                    for (int e = 0; e < VN; ++e)
                        if (gj0 + e < p.N) dst[e] = (p.r_zero ? T(0) : dst[e]) + val[e];
                }
            }
        }
    }
}

#undef COL
#undef STEP
#undef STEP_PLANES

// R[i][j] (+)= sum over splits s = 0..S-1 (ascending) of work[s][i][j].
// Work units are (row, 4 * blockDim-column chunk) pairs, so there is one
// integer division per unit instead of a 64-bit division per element (the
// per-element form cost ~15 us at 1024^2, about a third of it the divisions).
template <typename T>
__global__ void mmlt_splitk_reduce(const KParams p) {
    const int64_t total = p.M * p.N;
    const T* W = static_cast<const T*>(p.work);
    T* R = static_cast<T*>(p.R);
    const int64_t chunk = 4 * static_cast<int64_t>(blockDim.x);
    const int64_t per_row = (p.N + chunk - 1) / chunk;
    const int64_t units = p.M * per_row;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        int64_t i, j0;
        if (u <= 0xffffffffLL && per_row <= 0xffffffffLL) {  // a 32-bit division (the common case)
            const unsigned uu = static_cast<unsigned>(u), pr = static_cast<unsigned>(per_row);
            const unsigned i32 = uu / pr;
            i = i32;
            j0 = int64_t(uu - i32 * pr) * chunk;
        } else {
            i = u / per_row;
            j0 = (u - i * per_row) * chunk;
        }
        const int64_t j1 = j0 + chunk < p.N ? j0 + chunk : p.N;
        const T* w = W + i * p.N;
        T* r = R + i * p.ldr;
#pragma unroll 4
        for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
            T v = p.r_zero ? T(0) : r[j];
            for (int s = 0; s < p.splits; ++s) v = v + w[static_cast<int64_t>(s) * total + j];
            r[j] = v;
        }
    }
}

}  // namespace amltk

namespace amltk {

// Assignment statements (`R[i][j] = ...`): the reference's "last k wins"
// semantics (kernel_exec.cpp:299-312, test_exec.cpp:159-171) — only the
// k = k1-1 term reaches R. One thread per output element.
template <class Body, typename T>
__global__ void mmlt_assign_kernel(const KParams p) {
    const int64_t total = p.M * p.N;
    const T* A = static_cast<const T*>(p.A);
    const T* B = static_cast<const T*>(p.B);
    T* R = static_cast<T*>(p.R);
    const int64_t k = p.K - 1;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / p.N;
        const int64_t j = idx - i * p.N;
        typename Body::Acc acc[Body::NACC];
#pragma unroll
        for (int n = 0; n < Body::NACC; ++n) acc[n] = typename Body::Acc(0);
        const typename Body::Col c = (p.t_si || HasAt<Body>::value)
                                         ? col_at<Body, T>(Body::col(p, j), p, i, j)
                                         : Body::col(p, j);
        Body::step(acc, A[i * p.lda + k], B[k * p.ldb + j], c);
        R[i * p.ldr + j] = Body::finish(acc, c, 1);
    }
}

// Per-element executor for generated bodies (the naive run mode; the fixed
// bodies have theirs in naive.cu): one thread per R element, k ascending,
// `R += term` per k (or `R = term`), operands addressed through full strides.
struct NaiveStrides {
    int64_t sai, sak, sbk, sbj, sri, srj;
    int32_t accumulate;
};
template <class Body, typename T>
__global__ void mmlt_naive_body_kernel(const KParams p, const NaiveStrides s) {
    const int64_t total = p.M * p.N;
    const T* A = static_cast<const T*>(p.A);
    const T* B = static_cast<const T*>(p.B);
    T* R = static_cast<T*>(p.R);
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / p.N;
        const int64_t j = idx - i * p.N;
        const typename Body::Col c = col_at<Body, T>(Body::col(p, j), p, i, j);
        T* r = R + i * s.sri + j * s.srj;
        T acc = s.accumulate ? *r : T(0);
        for (int64_t k = 0; k < p.K; ++k) {
            const T v = Body::term(A[i * s.sai + k * s.sak], B[k * s.sbk + j * s.sbj], c);
            acc = s.accumulate ? add_rn(acc, v) : v;
        }
        if (p.K > 0 || s.accumulate) *r = acc;
    }
}

}  // namespace amltk
