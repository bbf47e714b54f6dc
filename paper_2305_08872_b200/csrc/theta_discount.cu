// theta_discount.cu — the discount body (preset q1, presets.cpp:66-67) in
// "theta form": one FP64-pipe compare and one DFMA per product instead of
// DMUL + DSETP + DFMA.
//
//   R[i][j] += sum_k  p * (p > t_j ? c1_j : 1),   p = rn(a_ik * b_kj),
//   c1_j = rn(1 - dis_j)
//
// For a fixed (k, j) the mask depends on a alone and is monotone in it:
// rn(x * b) is nondecreasing in x for b > 0 and nonincreasing for b < 0, so
// with
//   b > 0:  theta = max{ x : rn(x b) <= t }   mask  <=>  a > theta
//   b < 0:  theta = max{ x : rn(x b) >  t }   mask  <=>  !(a > theta)
// the mask is ONE compare of a against a per-(k, j) double, exactly (theta
// is found on the prepared side by a local walk from t/b and, failing that,
// bisection over the ordered bit patterns). The product then folds into the
// accumulate as acc = fma(a, P ? x1 : x0, acc) with
//   b > 0:  x0 = b,          x1 = rn(b c1)
//   b < 0:  x0 = rn(b c1),   x1 = b          (the compare sense flips)
//   b = 0:  x0 = x1 = b
// so the inner step is DSETP, 2 x SEL, DFMA (the shared a feeds both FP64
// instructions). B is prepared once per call into three planes (theta, x0,
// x1) of K x N doubles, staged per k tile by one 3-D TMA box.
//
// Results: the mask is exact, so integer-valued data (the reference's
// IntValued mode) is bit-exact; otherwise each term is a * rn(b c1) fused
// into the sum instead of rn(rn(a b) c1) added: a few ulps per term, inside
// BASELINE's 1e-12 f64 tolerance. The form is only equivalent when no product
// overflows or goes subnormal and every b, t, c1 is finite, so the prep and a
// per-run scan of A record the exponent ranges, and the theta kernel and an
// ordinary discount tile kernel (the fallback) are both launched: each reads
// the statistics and exactly one of them does the work. Non-finite a (inf,
// NaN) is handled by the theta form itself.
#include <cudaTypedefs.h>

#include <math_constants.h>

#include <cfloat>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "variants.h"

namespace amltk {
namespace th {

// Guard statistics (ints in the workspace header; zero = nothing seen).
// Exponents are stored biased so every slot is an atomicMax: max slots hold
// EB + e, min slots EB - e.
enum { G_BAD = 0, G_BMAX, G_BMIN, G_CMAX, G_CMIN, G_AMAX, G_AMIN, G_COUNT };
constexpr int EB = 4096;
constexpr int HEADER = 256;  // bytes before the planes

// floor(log2 |x|) for normal x; subnormal x reads as far out of range
__device__ __forceinline__ int expo(double x) {
    const int e = static_cast<int>((__double_as_longlong(x) >> 52) & 0x7ff);
    return e == 0 ? -1100 : e - 1023;
}

// The theta form is equivalent to the reference's evaluation when no term
// a b c1 can overflow or leave the normal range (|a b|, |a b c1| and |b c1|
// in [2^-1020, 2^1020]) and every b, t, c1 is finite.
__device__ __forceinline__ bool safe(const KParams& p) {
    const int* g = p.guard;
    if (g[G_BAD]) return false;
    auto mx = [&](int slot, int none) { return g[slot] ? g[slot] - EB : none; };
    auto mn = [&](int slot, int none) { return g[slot] ? EB - g[slot] : none; };
    const int hi = mx(G_AMAX, -1100) + mx(G_BMAX, -1100) + max(0, mx(G_CMAX, 0));
    const int lo = mn(G_AMIN, 0) + mn(G_BMIN, 0) + min(0, mn(G_CMIN, 0));
    return hi <= 1020 && lo >= -1020;
}

template <bool ROWS>
struct BodyThetaT {
    using Acc = double;
    static constexpr bool ROW_OUTER = ROWS;
    static constexpr int NACC = 1;
    static constexpr bool TWO_LEVEL = false;
    static constexpr int BPLANES = 3;
    static constexpr bool GUARDED = true;
    struct Col {};
    __device__ static Col col(const KParams&, int64_t) { return Col{}; }
    __device__ static __forceinline__ bool guard(const KParams& p) { return safe(p); }
    __device__ static __forceinline__ void step3(double* acc, double a, double theta, double x0, double x1) {
        acc[0] = fma_rn(a, a > theta ? x1 : x0, acc[0]);
    }
    __device__ static __forceinline__ double finish(const double* acc, const Col&, int64_t) { return acc[0]; }
};
using BodyTheta = BodyThetaT<false>;
using BodyThetaRows = BodyThetaT<true>;

// The ordinary discount tile kernel, run only when the theta form is not
// applicable to this call's operands.
struct BodyDiscountFallback : BodyDiscount<double> {
    static constexpr bool GUARDED = true;
    __device__ static __forceinline__ bool guard(const KParams& p) { return !safe(p); }
};

// Order-preserving int64 key of a non-NaN double (and back).
__device__ __forceinline__ long long okey(double x) {
    const long long b = __double_as_longlong(x);
    return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double odec(long long k) {
    return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL));
}
__device__ __forceinline__ bool pred(double x, double b, double t) {
    const double y = __dmul_rn(x, b);
    return b > 0 ? (y <= t) : (y > t);
}
// max{x : pred(x)}: pred is true-then-false over [-inf, +inf] (finite t,
// finite nonzero b), pred(-inf) holds and pred(+inf) does not.
// The walk steps over the ordered keys (one integer add per step instead of
// nextafter's special-case handling; -0 and +0 are adjacent keys with equal
// pred, so the maximum found is the same double up to the sign of a zero,
// which no compare a > theta can tell apart).
__device__ double theta_of(double b, double t) {
    double x = __dmul_rn(t, __drcp_rn(b));  // within ~2 ulps of t / b: the walk finishes it
    if (x != x) x = 0.0;
    long long kx = okey(x);
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
        if (!pred(odec(kx), b, t)) {
            --kx;
            continue;
        }
        if (!pred(odec(kx + 1), b, t)) return odec(kx);
        ++kx;
    }
    long long lo = okey(-CUDART_INF), hi = okey(CUDART_INF);
#pragma unroll 1
    while (static_cast<unsigned long long>(hi) - static_cast<unsigned long long>(lo) > 1ull) {
        const long long mid =
            lo + static_cast<long long>((static_cast<unsigned long long>(hi) - static_cast<unsigned long long>(lo)) >> 1);
        if (pred(odec(mid), b, t))
            lo = mid;
        else
            hi = mid;
    }
    return odec(lo);
}

// Block-wide max of up to G_COUNT slots, one atomicMax per slot per block.
template <int NS>
__device__ __forceinline__ void block_max(int (&v)[NS], int* g, int first) {
    __shared__ int red[NS][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int w = __reduce_max_sync(0xffffffffu, v[s]);
        if (lane == 0) red[s][warp] = w;
    }
    __syncthreads();
    if (threadIdx.x < NS) {
        int m = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = max(m, red[threadIdx.x][w]);
        if (m) atomicMax(g + first + threadIdx.x, m);
    }
}

// Units of the preparation and the A scan are (row, 4 * blockDim-column
// chunk) pairs: one integer division per unit, not a 64-bit division per
// element.
__device__ __forceinline__ void unit_of(int64_t u, int64_t per_row, int64_t cols, int64_t& row, int64_t& c0,
                                        int64_t& c1) {
    const int64_t chunk = 4 * static_cast<int64_t>(blockDim.x);
    if (u <= 0xffffffffLL && per_row <= 0xffffffffLL) {  // a 32-bit division (the common case)
        const unsigned uu = static_cast<unsigned>(u), pr = static_cast<unsigned>(per_row);
        const unsigned r32 = uu / pr;
        row = r32;
        c0 = int64_t(uu - r32 * pr) * chunk;
    } else {
        row = u / per_row;
        c0 = (u - row * per_row) * chunk;
    }
    c1 = c0 + chunk < cols ? c0 + chunk : cols;
}

// Planes (theta, x0, x1), each kdim x npad doubles, plus the B-side
// statistics, over blocks [0, nb) of the launch; this launch fills rows
// [plane_k0, plane_k0 + K) (planes points at row plane_k0 of the first
// plane).
__device__ __forceinline__ void prep_part(const KParams& p, double* planes, int64_t npad, int64_t pstride, int* g,
                                          int bid, int nb) {
    const double* B = static_cast<const double*>(p.B);
    const double* T = static_cast<const double*>(p.thres);
    const double* D = static_cast<const double*>(p.dis);
    int st[5] = {0, 0, 0, 0, 0};  // bad, bmax, bmin, cmax, cmin
    const int64_t per_row = (npad + 4 * blockDim.x - 1) / (4 * blockDim.x);
    for (int64_t u = bid; u < p.K * per_row; u += nb) {
        int64_t k, j0, j1;
        unit_of(u, per_row, npad, k, j0, j1);
        for (int64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
            double theta = 0.0, x0 = 0.0, x1 = 0.0;
            if (j < p.N) {
                const double b = B[k * p.ldb + j];
                const double t = T ? T[j * p.t_sj] : p.tconst;
                const double c1 = __dsub_rn(1.0, D[j * p.d_sj]);
                if (!isfinite(b) || !isfinite(t) || !isfinite(c1)) {
                    st[0] = 1;
                } else {
                    if (k == 0 && c1 != 0.0) {
                        const int e = expo(c1);
                        st[3] = max(st[3], EB + e);
                        st[4] = max(st[4], EB - e);
                    }
                    if (b == 0.0) {
                        x0 = x1 = b;
                    } else {
                        const int e = expo(b);
                        st[1] = max(st[1], EB + e);
                        st[2] = max(st[2], EB - e);
                        theta = theta_of(b, t);
                        const double bc = __dmul_rn(b, c1);
                        if (c1 != 0.0 && !(fabs(bc) >= DBL_MIN && fabs(bc) <= DBL_MAX)) st[0] = 1;
                        if (b > 0) {
                            x0 = b;
                            x1 = bc;
                        } else {
                            x0 = bc;
                            x1 = b;
                        }
                    }
                }
            }
            const int64_t idx = k * npad + j;
            planes[idx] = theta;
            planes[pstride + idx] = x0;
            planes[2 * pstride + idx] = x1;
        }
    }
    block_max<5>(st, g, G_BAD);
}

// A-side statistics of this run's rows (finite nonzero entries only), over
// blocks [0, nb).
__device__ __forceinline__ void a_stats_part(const KParams& p, int* g, int bid, int nb) {
    const double* A = static_cast<const double*>(p.A);
    int st[2] = {0, 0};
    const int64_t per_row = (p.K + 4 * blockDim.x - 1) / (4 * blockDim.x);
    for (int64_t u = bid; u < p.M * per_row; u += nb) {
        int64_t i, k0, k1;
        unit_of(u, per_row, p.K, i, k0, k1);
        double av[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // four loads in flight per thread
            const int64_t k = k0 + threadIdx.x + int64_t(q) * blockDim.x;
            av[q] = k < k1 ? __ldg(A + i * p.lda + k) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double a = av[q];
            if (a != 0.0 && isfinite(a)) {
                const int e = expo(a);
                st[0] = max(st[0], EB + e);
                st[1] = max(st[1], EB - e);
            }
        }
    }
    block_max<2>(st, g, G_AMAX);
}

// The preparation alone (panel-wise preparations; blocks [0, grid)) ...
__global__ void __launch_bounds__(256) prep_kernel(const KParams p, double* planes, int64_t npad, int64_t pstride,
                                                   int* g) {
    prep_part(p, planes, npad, pstride, g, blockIdx.x, gridDim.x);
}

// ... and, per call, the A scan, with the preparation of B in the same
// launch when it is not ready (blocks [0, nbp) prepare B, the rest scan A).
__global__ void __launch_bounds__(256) prep_stats_kernel(const KParams p, double* planes, int64_t npad,
                                                         int64_t pstride, int* g, int nbp) {
    if (static_cast<int>(blockIdx.x) < nbp)
        prep_part(p, planes, npad, pstride, g, blockIdx.x, nbp);
    else
        a_stats_part(p, g, blockIdx.x - nbp, gridDim.x - nbp);
}

int64_t npad_of(int64_t N) { return (N + 1) / 2 * 2; }  // 16-byte plane rows (TMA)

// blocks of 256 threads for the preparation / the A scan: one per unit, at
// most 16 per SM
// (at least one: an empty range still launches a valid grid)
int prep_blocks(const KParams& p) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(p.K * ((npad_of(p.N) + 1023) / 1024), 148 * 16)));
}
int a_stats_blocks(const KParams& p) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(p.M * ((p.K + 1023) / 1024), 148 * 8)));
}

// K rows of the preparation (panel-wise preparations: the whole K range)
int64_t kdim_of(const KParams& p) { return p.plane_kdim > 0 ? p.plane_kdim : p.K; }

size_t ws_bytes(const KParams& p) { return HEADER + size_t(3) * size_t(kdim_of(p)) * size_t(npad_of(p.N)) * 8; }

// B planes of k rows [plane_k0, plane_k0 + K). The statistics restart with
// the first panel (plane_k0 == 0) and accumulate over the later ones: a
// launch on panel p checks ranges over panels 0..p, a superset of its own.
cudaError_t prep_b(const KParams& p, void* ws, cudaStream_t s) {
    int* g = static_cast<int*>(ws);
    if (p.plane_k0 + p.K > kdim_of(p)) return cudaErrorInvalidValue;
    if (p.plane_k0 == 0) {
        const cudaError_t e = cudaMemsetAsync(g, 0, G_AMAX * sizeof(int), s);
        if (e != cudaSuccess) return e;
    }
    const int64_t npad = npad_of(p.N);
    const int64_t pstride = kdim_of(p) * npad;
    prep_kernel<<<prep_blocks(p), 256, 0, s>>>(
        p, reinterpret_cast<double*>(static_cast<char*>(ws) + HEADER) + p.plane_k0 * npad, npad, pstride, g);
    return cudaGetLastError();
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

bool encode(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box, bool swizzle128 = false) {
    auto fn = encoder();
    if (!fn) return false;
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// cudaFuncSetAttribute once per (kernel, device)
cudaError_t smem_attr_once(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kernel, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({kernel, dev});
    return e;
}

// the fallback's tile: the shipped discount f64 tile (32 x 128, 4 x 4 per thread)
constexpr int FB_TM = 4, FB_TN = 4, FB_WR = 8, FB_WC = 1, FB_BK = 16, FB_ST = 3, FB_MINB = 2;
using FbCfg = MmltTile<BodyDiscountFallback, double, FB_TM, FB_TN, FB_WR, FB_WC, FB_BK, FB_ST, LOAD_TMA, FB_MINB>;

template <class Body, int TM, int TN, int WR, int WC, int BK, int ST, int MINB, int LOAD>
cudaError_t run(const KParams& p, void* ws, bool b_ready, cudaStream_t s) {
    using Cfg = MmltTile<Body, double, TM, TN, WR, WC, BK, ST, LOAD, MINB>;
    int* g = static_cast<int*>(ws);
    const int64_t npad = npad_of(p.N);
    const double* planes = reinterpret_cast<const double*>(static_cast<char*>(ws) + HEADER) + p.plane_k0 * npad;
    cudaError_t e;
    // one reset and one launch: the B preparation (when not ready) and the
    // scan of this call's A rows side by side (the B-side statistics restart
    // with the first panel, plane_k0 == 0, and accumulate over later ones)
    {
        if (!b_ready && p.plane_k0 + p.K > kdim_of(p)) return cudaErrorInvalidValue;
        const bool reset_b = !b_ready && p.plane_k0 == 0;
        if ((e = cudaMemsetAsync(reset_b ? g : g + G_AMAX, 0, (reset_b ? G_COUNT : 2) * sizeof(int), s)) !=
            cudaSuccess)
            return e;
        const int nbp = b_ready ? 0 : prep_blocks(p);
        prep_stats_kernel<<<nbp + a_stats_blocks(p), 256, 0, s>>>(
            p, const_cast<double*>(planes), npad, kdim_of(p) * npad, g, nbp);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // theta kernel: A box BK x BM; B planes box BN x BK x 3
    CUtensorMap ma, mb;
    {
        const cuuint64_t ad[2] = {cuuint64_t(p.K), cuuint64_t(p.M)};
        const cuuint64_t as[1] = {cuuint64_t(p.lda) * 8};
        const cuuint32_t ab[2] = {cuuint32_t(BK), cuuint32_t(Cfg::BM)};
        const cuuint64_t bd[3] = {cuuint64_t(p.N), cuuint64_t(p.K), 3};
        const cuuint64_t bs[2] = {cuuint64_t(npad) * 8, cuuint64_t(kdim_of(p)) * cuuint64_t(npad) * 8};
        const cuuint32_t bb[3] = {cuuint32_t(Cfg::BN), cuuint32_t(BK), 3};
        if (!encode(&ma, p.A, 2, ad, as, ab, Cfg::SWZ) || !encode(&mb, planes, 3, bd, bs, bb))
            return cudaErrorInvalidValue;
    }
    // K segments (split-K): partials into p.work, reduced by the caller
    const int splits = p.splits > 1 && p.work ? p.splits : 1;
    KParams q = p;
    q.guard = g;
    q.splits = splits;
    q.kslice = splits > 1 ? p.kslice : p.K;
    q.work = splits > 1 ? p.work : nullptr;
    q.tiles_m = static_cast<int32_t>((p.M + Cfg::BM - 1) / Cfg::BM);
    q.tiles_n = static_cast<int32_t>((p.N + Cfg::BN - 1) / Cfg::BN);
    // raster groups of (resident CTAs / 8) row tiles, so one wave covers a
    // group's rows x about 8 column panels: DRAM reads of 4096 rows of config
    // 4 fall from 92.6 GB (512-row groups) to 56.9 GB at the same speed
    // (tools/raster_probe.sh; 960 / 3552-row groups read 66.3 / 68.2 GB)
    q.group_m = std::min(64, std::max(8, 148 * MINB / 8));
    if (const char* gr = getenv("AMLT_THETA_GROUP_ROWS"))  // raster experiments (tools/raster_probe.sh)
        q.group_m = std::max(1, atoi(gr) / Cfg::BM);
    auto kt = &mmlt_tile_kernel<Body, double, TM, TN, WR, WC, BK, ST, LOAD, MINB>;
    if ((e = smem_attr_once(reinterpret_cast<const void*>(kt), Cfg::SMEM_BYTES)) != cudaSuccess) return e;
    kt<<<dim3(static_cast<unsigned>(int64_t(q.tiles_m) * q.tiles_n), static_cast<unsigned>(splits)), Cfg::THREADS,
         Cfg::SMEM_BYTES, s>>>(q, ma, mb);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    // fallback: the ordinary discount tile over the raw operands
    CUtensorMap fa, fb;
    {
        const cuuint64_t ad[2] = {cuuint64_t(p.K), cuuint64_t(p.M)};
        const cuuint64_t as[1] = {cuuint64_t(p.lda) * 8};
        const cuuint32_t ab[2] = {cuuint32_t(FB_BK), cuuint32_t(FbCfg::BM)};
        const cuuint64_t bd[2] = {cuuint64_t(p.N), cuuint64_t(p.K)};
        const cuuint64_t bs[1] = {cuuint64_t(p.ldb) * 8};
        const cuuint32_t bb[2] = {cuuint32_t(FbCfg::BN), cuuint32_t(FB_BK)};
        if (!encode(&fa, p.A, 2, ad, as, ab) || !encode(&fb, p.B, 2, bd, bs, bb)) return cudaErrorInvalidValue;
    }
    KParams f = q;
    f.tiles_m = static_cast<int32_t>((p.M + FbCfg::BM - 1) / FbCfg::BM);
    f.tiles_n = static_cast<int32_t>((p.N + FbCfg::BN - 1) / FbCfg::BN);
    f.group_m = std::min(64, std::max(8, 512 / FbCfg::BM));
    auto kf = &mmlt_tile_kernel<BodyDiscountFallback, double, FB_TM, FB_TN, FB_WR, FB_WC, FB_BK, FB_ST, LOAD_TMA,
                                FB_MINB>;
    if ((e = smem_attr_once(reinterpret_cast<const void*>(kf), FbCfg::SMEM_BYTES)) != cudaSuccess) return e;
    kf<<<dim3(static_cast<unsigned>(int64_t(f.tiles_m) * f.tiles_n), static_cast<unsigned>(splits)), FbCfg::THREADS,
         FbCfg::SMEM_BYTES, s>>>(f, fa, fb);
    return cudaGetLastError();
}

cudaError_t no_tile_launch(const KParams&, const CUtensorMap&, const CUtensorMap&, dim3, cudaStream_t) {
    return cudaErrorNotSupported;  // launched through VariantDesc::run
}

}  // namespace th

template <int TM, int TN, int WR, int WC, int BK, int ST, int MINB, int LOAD = LOAD_TMA, class Body = th::BodyTheta>
void add_theta(Registry& reg, const char* name) {
    using Cfg = MmltTile<Body, double, TM, TN, WR, WC, BK, ST, LOAD, MINB>;
    VariantDesc v;
    v.body = 1;   // AMLT_BODY_DISCOUNT
    v.dtype = 0;  // AMLT_F64
    v.bm = Cfg::BM;
    v.bn = Cfg::BN;
    v.bk = BK;
    v.tm = TM;
    v.tn = TN;
    v.threads = Cfg::THREADS;
    v.stages = ST;
    v.smem = Cfg::SMEM_BYTES;
    v.minb = MINB;
    v.vec = true;
    v.name = name;
    v.func = reinterpret_cast<const void*>(
        &mmlt_tile_kernel<Body, double, TM, TN, WR, WC, BK, ST, LOAD, MINB>);
    v.launch = &th::no_tile_launch;
    v.ws_bytes = &th::ws_bytes;
    v.run = &th::run<Body, TM, TN, WR, WC, BK, ST, MINB, LOAD>;
    v.prep_b = &th::prep_b;
    v.prep_id = 3;  // (theta, x0, x1) planes of B, shared by every theta tile
    v.splittable = true;
    v.prep_panels = true;
    v.r_overwrite = true;  // the tile kernel's epilogue (theta and fallback)
    reg.variants.push_back(v);
}

void register_theta_discount(Registry& reg) {
    // 8 x 4 micro-tiles take 150+ registers (one CTA per SM; the 96-row tile
    // runs 12 warps), 6 x 4 ones 126 (two 8-warp CTAs per SM: 16 warps)
    //                 TM TN WR WC BK ST MINB
    add_theta<4, 4, 8, 1, 8, 4, 2>(reg, "theta_t4x4_w8x1");
    add_theta<8, 2, 8, 1, 16, 3, 2>(reg, "theta_t8x2_w8x1");
    add_theta<8, 4, 8, 1, 16, 3, 1>(reg, "theta_t8x4_w8x1");
    add_theta<8, 4, 4, 2, 16, 2, 1>(reg, "theta_t8x4_w4x2");
    add_theta<8, 4, 12, 1, 16, 2, 1>(reg, "theta_t8x4_w12x1");
    add_theta<6, 4, 8, 1, 16, 2, 2>(reg, "theta_t6x4_w8x1");
    // A 2-D lane grid (4 lanes along rows, 8 along columns): a third of the
    // shared-memory wavefronts per product. Measured slower than the 1 x 32
    // grids at 8192^3 (100.9 vs 98.9 ms; shared-memory bandwidth is not what
    // bounds this body, profiles/r01/thetabench.txt); kept as a tuner
    // candidate and to keep the lane-grid path exercised.
    add_theta<8, 4, 3, 4, 16, 2, 1, LOAD_TMA | LOAD_LR4>(reg, "theta_t8x4_l4x8_w3x4");
    // 16 warps per SM (4 per scheduler) with 6 rows per thread. Measured at
    // 8192^3 (tools/quick_perf.py, r02): 99.8 ms against 98.8 for the 12-warp
    // 8 x 4 tile; 5 x 4 (101.4), 6 x 4 BK = 8 (100.1) and row-outer inner
    // order (104.7) were slower and are not kept; so was (r02) a 20-warp
    // 4 x 4 tile on the lane grid in 64 x 32 CTAs, five per SM (118.6 ms:
    // 96 registers with small spills, and a third more loads per product).
    add_theta<6, 4, 16, 1, 16, 2, 1>(reg, "theta_t6x4_w16x1");
}

}  // namespace amltk
