// swar_eqcount.cu — the equality-count body (`R[i][j] += A[i][k] == B[k][j]`,
// int32; eqcmp, maskadd, add) four products at a time.
//
// When every value of A and B lies in one window of 128 consecutive
// integers, v -> v mod 128 is injective on the window, so equality of two
// values is equality of their low 7 bits. A pre-pass packs four consecutive
// k of A (per row) and of B (per column) into one 32-bit word of 7-bit bytes;
// then for a packed pair (a4, b4)
//
//     x = a4 ^ b4                         bytes are 0 exactly where equal
//     y = (x + 0x7F7F7F7F) & 0x80808080   0x80 in each differing byte (no
//                                         carry crosses a byte: 0x7F + 0x7F)
//     n += y >> 7                         per-byte counters (mad.hi, one op)
//
// four ALU instructions for four products, against SETP + predicated add
// per product for the plain body: 0.898 ms against 1.110 at config 3b's shape
// (65536 x 256 x 1024, A and B uniform 0..15), packing included. The byte counters hold at most BK per k tile;
// the tile kernel's two-level accumulation folds them into a full int per
// tile (Body::fold). The count is of DIFFERING pairs, so the padding of K to
// whole words (A pads with 0, B with 1) counts as different and the result
// is 4 * words - n.
//
// The window check is data-dependent: the pre-passes record min and max of
// A and B, and the packed kernel and the ordinary eqcount tile (over the raw
// operands) are both launched; each reads the statistics at CTA start and
// exactly one of them does the work (as the theta-form discount does).
// Results are exact integers either way.
#include <cudaTypedefs.h>

#include <climits>
#include <mutex>
#include <set>
#include <utility>

#include "variants.h"

namespace amltk {
namespace sw {

// Header words: min / max of B (prepared once per call), min / max of A (per
// run), as order-preserving unsigned keys v ^ 0x80000000, so the sentinels
// are plain byte fills (0xFF.. for min, 0 for max) below / above any value.
enum { G_BMIN = 0, G_BMAX, G_AMIN, G_AMAX };
__host__ __device__ __forceinline__ unsigned okey32(int v) { return static_cast<unsigned>(v) ^ 0x80000000u; }
constexpr int HEADER = 256;  // bytes before the packed operands

__device__ __forceinline__ bool window_ok(const KParams& p) {
    const unsigned* g = reinterpret_cast<const unsigned*>(p.guard);
    const unsigned mn = min(g[G_BMIN], g[G_AMIN]), mx = max(g[G_BMAX], g[G_AMAX]);
    return mx < mn || mx - mn <= 127u;  // (mx < mn: no elements)
}

// (Moving the add or the count onto the FMA pipe as integer multiply-adds
// with run-time multipliers measured slower: 0.916 / 1.016 ms against 0.898
// at config 3b's shape, so all four stay ALU instructions.)
struct BodySwarEq {
    using Acc = int;
    static constexpr int NACC = 1;
    static constexpr bool TWO_LEVEL = true;  // byte-lane partials per k tile
    static constexpr bool FOLD = true;
    static constexpr bool GUARDED = true;
    struct Col {};
    __device__ static Col col(const KParams&, int64_t) { return {}; }
    __device__ static __forceinline__ bool guard(const KParams& p) { return window_ok(p); }
    __device__ static __forceinline__ void step(int* acc, int a4, int b4, const Col&) {
        const unsigned x = static_cast<unsigned>(a4) ^ static_cast<unsigned>(b4);
        const unsigned y = (x + 0x7F7F7F7Fu) & 0x80808080u;
        asm("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc[0]) : "r"(y), "r"(1u << 25));
    }
    __device__ static __forceinline__ void fold(int& acc, const int& part) {
        const unsigned u = static_cast<unsigned>(part);
        acc += static_cast<int>((u & 0xFFu) + ((u >> 8) & 0xFFu) + ((u >> 16) & 0xFFu) + (u >> 24));
    }
    // kwords: packed words of the k range, padding included
    __device__ static __forceinline__ int finish(const int* acc, const Col&, int64_t kwords) {
        return static_cast<int>(4 * kwords) - acc[0];
    }
};

// the ordinary eqcount tile over the raw operands, when the window check fails
struct BodyEqFallback : BodyEqcount<int> {
    static constexpr bool GUARDED = true;
    __device__ static __forceinline__ bool guard(const KParams& p) { return !window_ok(p); }
};

int64_t kw_of(int64_t K) { return ((K + 3) / 4 + 3) / 4 * 4; }  // words per packed row (16-byte pitch)
int64_t npad_of(int64_t N) { return (N + 3) / 4 * 4; }

__device__ __forceinline__ void block_minmax(unsigned mn, unsigned mx, int* gi, int slot_min) {
    unsigned* g = reinterpret_cast<unsigned*>(gi);
    __shared__ unsigned red[2][8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    mn = __reduce_min_sync(0xffffffffu, mn);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
        red[0][warp] = mn;
        red[1][warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            mn = min(mn, red[0][w]);
            mx = max(mx, red[1][w]);
        }
        if (mn != 0xFFFFFFFFu) atomicMin(g + slot_min, mn);
        if (mx != 0u) atomicMax(g + slot_min + 1, mx);
    }
}

// B4[w][j] = bytes (B[4w + e][j] & 0x7F), e = 0..3; 1 past K
__global__ void __launch_bounds__(256) pack_b_kernel(const KParams p, unsigned* B4, int64_t kw, int64_t npad,
                                                     int* g) {
    const int* B = static_cast<const int*>(p.B);
    unsigned mn = 0xFFFFFFFFu, mx = 0u;
    const int64_t total = kw * npad;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t w = idx / npad, j = idx - w * npad;
        unsigned word = 0;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int64_t k = 4 * w + e;
            unsigned byte = 1u;
            if (k < p.K && j < p.N) {
                const int v = B[k * p.ldb + j];
                mn = min(mn, okey32(v));
                mx = max(mx, okey32(v));
                byte = static_cast<unsigned>(v) & 0x7Fu;
            }
            word |= byte << (8 * e);
        }
        B4[idx] = word;
    }
    block_minmax(mn, mx, g, G_BMIN);
}

// A4[i][w] = bytes (A[i][4w + e] & 0x7F); 0 past K
__global__ void __launch_bounds__(256) pack_a_kernel(const KParams p, unsigned* A4, int64_t kw, int* g) {
    const int* A = static_cast<const int*>(p.A);
    unsigned mn = 0xFFFFFFFFu, mx = 0u;
    const int64_t total = p.M * kw;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = idx / kw, w = idx - i * kw;
        unsigned word = 0;
        if (4 * w + 3 < p.K) {  // one 16-byte load (the variants take 16-byte aligned operands)
            const int4 v = *reinterpret_cast<const int4*>(A + i * p.lda + 4 * w);
            mn = min(mn, okey32(min(min(v.x, v.y), min(v.z, v.w))));
            mx = max(mx, okey32(max(max(v.x, v.y), max(v.z, v.w))));
            word = (static_cast<unsigned>(v.x) & 0x7Fu) | ((static_cast<unsigned>(v.y) & 0x7Fu) << 8) |
                   ((static_cast<unsigned>(v.z) & 0x7Fu) << 16) | ((static_cast<unsigned>(v.w) & 0x7Fu) << 24);
        } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t k = 4 * w + e;
                if (k < p.K) {
                    const int v = A[i * p.lda + k];
                    mn = min(mn, okey32(v));
                    mx = max(mx, okey32(v));
                    word |= (static_cast<unsigned>(v) & 0x7Fu) << (8 * e);
                }
            }
        }
        A4[idx] = word;
    }
    block_minmax(mn, mx, g, G_AMIN);
}

size_t b_bytes(const KParams& p) { return size_t(kw_of(p.K)) * size_t(npad_of(p.N)) * 4; }
size_t ws_bytes(const KParams& p) { return HEADER + b_bytes(p) + size_t(p.M) * size_t(kw_of(p.K)) * 4; }

// min slot starts at the largest key, max slot at the smallest
cudaError_t reset_stats(int* g, int slot_min, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(g + slot_min, 0xFF, sizeof(int), s);
    if (e == cudaSuccess) e = cudaMemsetAsync(g + slot_min + 1, 0x00, sizeof(int), s);
    return e;
}

cudaError_t prep_b(const KParams& p, void* ws, cudaStream_t s) {
    int* g = static_cast<int*>(ws);
    cudaError_t e = reset_stats(g, G_BMIN, s);
    if (e != cudaSuccess) return e;
    const int64_t kw = kw_of(p.K), npad = npad_of(p.N);
    const int blocks = static_cast<int>(std::min<int64_t>((kw * npad + 255) / 256, 148 * 16));
    pack_b_kernel<<<blocks, 256, 0, s>>>(p, reinterpret_cast<unsigned*>(static_cast<char*>(ws) + HEADER), kw,
                                         npad, g);
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

// 2-D int32 map: inner x outer elements, row pitch in elements, box bi x bo
bool encode(CUtensorMap* m, const void* base, int64_t inner, int64_t outer, int64_t pitch, int bi, int bo) {
    auto fn = encoder();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
    const cuuint64_t strides[1] = {cuuint64_t(pitch) * 4};
    const cuuint32_t box[2] = {cuuint32_t(bi), cuuint32_t(bo)};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

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

// the fallback's tile: the ordinary i32 eqcount tile (32 x 128, 4 x 4 per thread)
constexpr int FB_TM = 4, FB_TN = 4, FB_WR = 8, FB_WC = 1, FB_BK = 32, FB_ST = 3, FB_MINB = 2;
using FbCfg = MmltTile<BodyEqFallback, int, FB_TM, FB_TN, FB_WR, FB_WC, FB_BK, FB_ST, LOAD_TMA, FB_MINB>;

template <int TM, int TN, int WR, int WC, int BK, int ST, int MINB>
cudaError_t run(const KParams& p, void* ws, bool b_ready, cudaStream_t s) {
    using Cfg = MmltTile<BodySwarEq, int, TM, TN, WR, WC, BK, ST, LOAD_TMA, MINB>;
    static_assert(BK <= 255, "byte-lane partials must not overflow within a k tile");
    int* g = static_cast<int*>(ws);
    const int64_t kw = kw_of(p.K), npad = npad_of(p.N);
    unsigned* B4 = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + HEADER);
    unsigned* A4 = reinterpret_cast<unsigned*>(static_cast<char*>(ws) + HEADER + b_bytes(p));
    cudaError_t e;
    if (!b_ready && (e = prep_b(p, ws, s)) != cudaSuccess) return e;
    if ((e = reset_stats(g, G_AMIN, s)) != cudaSuccess) return e;
    {
        const int blocks = static_cast<int>(std::min<int64_t>((p.M * kw + 255) / 256, 148 * 16));
        pack_a_kernel<<<blocks, 256, 0, s>>>(p, A4, kw, g);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // packed kernel over K' = kw words
    CUtensorMap ma, mb;
    if (!encode(&ma, A4, kw, p.M, kw, BK, Cfg::BM) || !encode(&mb, B4, p.N, kw, npad, Cfg::BN, BK))
        return cudaErrorInvalidValue;
    KParams q = p;
    q.A = A4;
    q.lda = kw;
    q.B = B4;
    q.ldb = npad;
    q.K = kw;
    q.kslice = kw;
    q.splits = 1;
    q.work = nullptr;
    q.guard = g;
    q.tiles_m = static_cast<int32_t>((p.M + Cfg::BM - 1) / Cfg::BM);
    q.tiles_n = static_cast<int32_t>((p.N + Cfg::BN - 1) / Cfg::BN);
    q.group_m = std::min(64, std::max(8, 512 / Cfg::BM));
    auto kt = &mmlt_tile_kernel<BodySwarEq, int, TM, TN, WR, WC, BK, ST, LOAD_TMA, MINB>;
    if ((e = smem_attr_once(reinterpret_cast<const void*>(kt), Cfg::SMEM_BYTES)) != cudaSuccess) return e;
    kt<<<static_cast<unsigned>(int64_t(q.tiles_m) * q.tiles_n), Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(q, ma, mb);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;

    // fallback: the ordinary eqcount tile over the raw operands
    CUtensorMap fa, fb;
    if (!encode(&fa, p.A, p.K, p.M, p.lda, FB_BK, FbCfg::BM) || !encode(&fb, p.B, p.N, p.K, p.ldb, FbCfg::BN, FB_BK))
        return cudaErrorInvalidValue;
    KParams f = p;
    f.guard = g;
    f.splits = 1;
    f.kslice = p.K;
    f.work = nullptr;
    f.tiles_m = static_cast<int32_t>((p.M + FbCfg::BM - 1) / FbCfg::BM);
    f.tiles_n = static_cast<int32_t>((p.N + FbCfg::BN - 1) / FbCfg::BN);
    f.group_m = std::min(64, std::max(8, 512 / FbCfg::BM));
    auto kf = &mmlt_tile_kernel<BodyEqFallback, int, FB_TM, FB_TN, FB_WR, FB_WC, FB_BK, FB_ST, LOAD_TMA, FB_MINB>;
    if ((e = smem_attr_once(reinterpret_cast<const void*>(kf), FbCfg::SMEM_BYTES)) != cudaSuccess) return e;
    kf<<<static_cast<unsigned>(int64_t(f.tiles_m) * f.tiles_n), FbCfg::THREADS, FbCfg::SMEM_BYTES, s>>>(f, fa, fb);
    return cudaGetLastError();
}

cudaError_t no_tile_launch(const KParams&, const CUtensorMap&, const CUtensorMap&, dim3, cudaStream_t) {
    return cudaErrorNotSupported;  // launched through VariantDesc::run
}

}  // namespace sw

template <int TM, int TN, int WR, int WC, int BK, int ST, int MINB>
void add_swar(Registry& reg, const char* name) {
    using Cfg = MmltTile<sw::BodySwarEq, int, TM, TN, WR, WC, BK, ST, LOAD_TMA, MINB>;
    VariantDesc v;
    v.body = 4;   // AMLT_BODY_EQCOUNT
    v.dtype = 2;  // AMLT_I32
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
        &mmlt_tile_kernel<sw::BodySwarEq, int, TM, TN, WR, WC, BK, ST, LOAD_TMA, MINB>);
    v.launch = &sw::no_tile_launch;
    v.ws_bytes = &sw::ws_bytes;
    v.run = &sw::run<TM, TN, WR, WC, BK, ST, MINB>;
    v.r_overwrite = true;  // packed and fallback launches are both the tile kernel
    v.prep_b = &sw::prep_b;
    v.prep_id = 6;  // 7-bit byte-packed B
    reg.variants.push_back(v);
}

void register_swar_eqcount(Registry& reg) {
    //        TM TN WR WC BK ST MINB
    add_swar<4, 4, 8, 1, 32, 3, 2>(reg, "swar_t4x4_w8x1");
    add_swar<8, 4, 8, 1, 32, 3, 1>(reg, "swar_t8x4_w8x1");
    add_swar<4, 4, 4, 1, 32, 4, 3>(reg, "swar_t4x4_w4x1");
    add_swar<4, 8, 8, 1, 32, 3, 1>(reg, "swar_t4x8_w8x1");
}

}  // namespace amltk
