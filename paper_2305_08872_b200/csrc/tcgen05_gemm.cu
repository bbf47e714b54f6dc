// tcgen05_gemm.cu — the plain-GEMM body in f32 on the 5th-generation tensor
// cores: tcgen05.mma kind::tf32 with a 3xTF32 split.
//
//   R[i][j] += sum_k A[i][k] * B[k][j]        (preset matmul, presets.cpp:64-65)
//
// A TF32 product alone would miss BASELINE's 1e-5 (fp32 vs the fp64 oracle),
// so every operand is split into two TF32-representable parts, x = x_hi +
// x_lo (x_hi = x rounded to 11 significant bits, x_lo = x - x_hi rounded the
// same way), and
//     A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi
// (the dropped A_lo B_lo term and the rounding of x_lo are ~2^-22 relative:
// FFMA-class accuracy). The three products are one TF32 GEMM over a K three
// times as deep: a pre-pass writes A' = [A_hi | A_hi | A_lo] (M x 3K, K
// contiguous) and B'^T = [B_hi | B_lo | B_hi]^T (N x 3K, K contiguous) into
// the context workspace, so both operands are K-major for the tensor core.
//
// The GEMM is the canonical sm_100a structure (one CTA per 128 x 128 tile,
// 192 threads, warp-specialised):
//   warp 0, one lane   TMA producer: 6-stage ring of A' (32 x 128) and B'^T
//                      (32 x 128) boxes, 128-byte swizzle, full/empty
//                      mbarriers;
//   warp 1             allocates all 512 TMEM columns: four 128 x 128 fp32
//                      accumulators that take the k blocks round-robin; one
//                      lane issues tcgen05.mma (M=128, N=128, K=8) x 4 per
//                      stage and tcgen05.commit frees the stage / signals the
//                      epilogue;
//   warps 2-5          epilogue: tcgen05.ld 32 lanes x 16 columns at a time
//                      from each accumulator, summed with IEEE adds, then
//                      R += sum (fp32).
// Integer-valued inputs split exactly (x_lo = 0), so the int-valued parity
// cases stay bit-exact.
#include <cudaTypedefs.h>

#include <mutex>

#include "variants.h"

namespace amltk {
namespace tc {

constexpr int BM = 128, BK = 32, UMMA_K = 8;
constexpr int THREADS = 192;
constexpr int STAGE_A = BM * BK * 4;  // bytes per stage

// Tile width, accumulator count and ring depth. The tensor core's fp32
// accumulation loses more than IEEE adds over long chains, so k blocks go
// round-robin to NACC independent TMEM accumulators (each chain NACC times
// shorter), summed by the epilogue with IEEE adds; NACC x BN = 512 columns,
// the whole TMEM of the SM.
template <int BN_, int NACC_, int STAGES_>
struct TcCfg {
    static constexpr int BN = BN_, NACC = NACC_, STAGES = STAGES_;
    static constexpr int STAGE_B = BN * BK * 4;
    static constexpr int SMEM = STAGES * (STAGE_A + STAGE_B) + 1024 + 256;  // + alignment + barriers
    static constexpr uint32_t TMEM_COLS = NACC * BN;
    // kind::tf32, fp32 accumulate, A and B K-major, M = BM, N = BN
    static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN >> 3) << 17) |
                                      (uint32_t(BM >> 4) << 24);
    static_assert(NACC * BN <= 512, "TMEM holds 512 fp32 columns");
    static_assert(STAGES * (STAGE_A + STAGE_B) + 1280 <= 232448, "shared memory");
};
using Wide = TcCfg<256, 2, 4>;    // 128 x 256 tiles
using Narrow = TcCfg<128, 4, 6>;  // 128 x 128 tiles, shorter accumulation chains

struct TcParams {
    float* R;
    int64_t ldr;
    int64_t M, N, K3;
    int32_t tiles_m, tiles_n, group_m;
    int32_t r_vec_ok;
};

__device__ __forceinline__ float tf32_round(float x) {
    // round to 11 significant bits (nearest, ties away from zero); a finite x
    // that would round up to infinity is truncated instead, inf / nan pass
    const uint32_t u = __float_as_uint(x);
    uint32_t r = (u + 0x1000u) & 0xFFFFE000u;
    if ((r & 0x7F800000u) == 0x7F800000u && (u & 0x7F800000u) != 0x7F800000u) r = u & 0xFFFFE000u;
    return __uint_as_float(r);
}

// A' row i = [hi(A[i][:]) | hi(A[i][:]) | lo(A[i][:])]
__global__ void split_a_kernel(const float* __restrict__ A, int64_t lda, int64_t M, int64_t K,
                               float* __restrict__ Ap, int64_t ld3) {
    const int64_t total = M * K;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = idx / K, k = idx - i * K;
        const float a = A[i * lda + k];
        const float hi = tf32_round(a);
        const float lo = tf32_round(a - hi);
        float* row = Ap + i * ld3;
        row[k] = hi;
        row[K + k] = hi;
        row[2 * K + k] = lo;
    }
}

// B'^T row j = [hi(B[:][j]) | lo(B[:][j]) | hi(B[:][j])]: a 32 x 32 smem
// transpose (coalesced reads along j, writes along k)
__global__ void split_bt_kernel(const float* __restrict__ B, int64_t ldb, int64_t K, int64_t N,
                                float* __restrict__ Bt, int64_t ld3) {
    __shared__ float tile[32][33];
    const int64_t k0 = int64_t(blockIdx.y) * 32, j0 = int64_t(blockIdx.x) * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t k = k0 + r, j = j0 + threadIdx.x;
        tile[r][threadIdx.x] = (k < K && j < N) ? B[k * ldb + j] : 0.f;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int64_t j = j0 + r, k = k0 + threadIdx.x;
        if (j < N && k < K) {
            const float b = tile[threadIdx.x][r];
            const float hi = tf32_round(b);
            const float lo = tf32_round(b - hi);
            float* row = Bt + j * ld3;
            row[k] = hi;
            row[K + k] = lo;
            row[2 * K + k] = hi;
        }
    }
}

// ---- PTX wrappers (tcgen05 / TMA / mbarrier)

__device__ __forceinline__ uint32_t su32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(su32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int32_t x, int32_t y,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
// K-major operand tile in 128-byte-swizzled rows (8-row atoms 1024 B apart)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= uint64_t((addr & 0x3FFFF) >> 4);  // start address
    d |= uint64_t(1) << 16;                // leading byte offset (unused for swizzled K-major)
    d |= uint64_t(1024 >> 4) << 32;        // stride byte offset: next 8-row atom
    d |= uint64_t(1) << 46;                // descriptor version (sm_100)
    d |= uint64_t(2) << 61;                // SWIZZLE_128B
    return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     su32(bar))
                 : "memory");
}

template <class Cfg>
__global__ void __launch_bounds__(THREADS, 1)
    tf32x3_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                       const TcParams p) {
    constexpr int BN = Cfg::BN, NACC = Cfg::NACC, STAGES = Cfg::STAGES, STAGE_B = Cfg::STAGE_B;
    constexpr uint32_t TMEM_COLS = Cfg::TMEM_COLS;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = base;
    unsigned char* sB = base + STAGES * STAGE_A;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * STAGE_B);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    // grouped raster (L2 reuse of B' panels across the group's row tiles)
    const int G = p.group_m, bid = blockIdx.x, per_group = G * p.tiles_n;
    const int group = bid / per_group, first_m = group * G;
    const int gsize = min(p.tiles_m - first_m, G), in_group = bid - group * per_group;
    const int64_t m0 = int64_t(first_m + in_group % gsize) * BM;
    const int64_t n0 = int64_t(in_group / gsize) * BN;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nkb = static_cast<int>((p.K3 + BK - 1) / BK);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            bar_init(&full[s], 1);
            bar_init(&empty[s], 1);
        }
        bar_init(acc_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         su32(tmem_slot)),
                     "r"(TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % STAGES;
                bar_wait(&empty[s], ((kb / STAGES) & 1) ^ 1);
                bar_expect(&full[s], STAGE_A + STAGE_B);
                tma_2d(sA + s * STAGE_A, &tmA, kb * BK, static_cast<int32_t>(m0), &full[s]);
                tma_2d(sB + s * STAGE_B, &tmB, kb * BK, static_cast<int32_t>(n0), &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % STAGES;
                bar_wait(&full[s], (kb / STAGES) & 1);
                fence_after();
                const uint32_t a0 = su32(sA + s * STAGE_A), b0 = su32(sB + s * STAGE_B);
                const uint32_t acc = tmem + uint32_t((kb % NACC) * BN);
#pragma unroll
                for (int k = 0; k < BK / UMMA_K; ++k)
                    mma_tf32(acc, smem_desc(a0 + k * UMMA_K * 4), smem_desc(b0 + k * UMMA_K * 4),
                             Cfg::IDESC, (kb >= NACC) || k != 0);
                mma_commit(&empty[s]);  // frees the stage once these MMAs have read it
            }
            mma_commit(acc_full);  // accumulator complete
        }
    } else {  // epilogue warps 2..5: TMEM lane quarter (warp % 4)
        bar_wait(acc_full, 0);
        fence_after();
        const int q = warp & 3;
        const int64_t row = m0 + 32 * q + lane;
        const int used = nkb < NACC ? nkb : NACC;  // accumulators that received k blocks
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
            float sum[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) sum[e] = 0.f;
#pragma unroll 1
            for (int a = 0; a < used; ++a) {
                uint32_t v[16];
                const uint32_t taddr = tmem + (uint32_t(32 * q) << 16) + uint32_t(a * BN + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, "
                    "%10, %11, %12, %13, %14, %15}, [%16];\n"
                    : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                      "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
                      "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                    : "r"(taddr));
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int e = 0; e < 16; ++e) sum[e] = __fadd_rn(sum[e], __uint_as_float(v[e]));
            }
            if (row < p.M) {
                const int64_t col = n0 + c0;
                float* dst = p.R + row * p.ldr + col;
                if (p.r_vec_ok && col + 16 <= p.N) {
#pragma unroll
                    for (int e = 0; e < 16; e += 4) {
                        float4 o = *reinterpret_cast<float4*>(dst + e);
                        o.x += sum[e];
                        o.y += sum[e + 1];
                        o.z += sum[e + 2];
                        o.w += sum[e + 3];
                        *reinterpret_cast<float4*>(dst + e) = o;
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (col + e < p.N) dst[e] += sum[e];
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TMEM_COLS));
}

// ---- host side

int64_t ld3_of(int64_t K) { return (3 * K + 3) / 4 * 4; }  // 16-byte row pitch (TMA)

// Workspace: B'^T first (the part shared by every row band of one call),
// then A'.
size_t b_bytes(const KParams& p) { return (size_t(p.N) * ld3_of(p.K) * 4 + 255) / 256 * 256; }
size_t ws_bytes(const KParams& p) { return b_bytes(p) + size_t(p.M) * ld3_of(p.K) * 4 + 256; }

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

bool encode(CUtensorMap* m, const float* base, int64_t inner, int64_t outer, int64_t ld, int box_outer) {
    auto fn = encoder();
    if (!fn) return false;
    cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 4};
    cuuint32_t box[2] = {cuuint32_t(BK), cuuint32_t(box_outer)};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t prep_b(const KParams& p, void* ws, cudaStream_t s) {
    const int64_t N = p.N, K = p.K, ld3 = ld3_of(K);
    float* Bt = static_cast<float*>(ws);
    dim3 g(static_cast<unsigned>((N + 31) / 32), static_cast<unsigned>((K + 31) / 32));
    split_bt_kernel<<<g, dim3(32, 8), 0, s>>>(static_cast<const float*>(p.B), p.ldb, K, N, Bt, ld3);
    return cudaGetLastError();
}

template <class Cfg>
cudaError_t run(const KParams& p, void* ws, bool b_ready, cudaStream_t s) {
    constexpr int BN = Cfg::BN;
    const int64_t M = p.M, N = p.N, K = p.K, ld3 = ld3_of(K);
    float* Bt = static_cast<float*>(ws);
    float* Ap = reinterpret_cast<float*>(static_cast<char*>(ws) + b_bytes(p));
    if (!b_ready) {
        const cudaError_t e = prep_b(p, ws, s);
        if (e != cudaSuccess) return e;
    }
    {
        const int64_t total = M * K;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 32));
        split_a_kernel<<<blocks, 256, 0, s>>>(static_cast<const float*>(p.A), p.lda, M, K, Ap, ld3);
    }
    CUtensorMap ma, mb;
    if (!encode(&ma, Ap, 3 * K, M, ld3, BM) || !encode(&mb, Bt, 3 * K, N, ld3, BN))
        return cudaErrorInvalidValue;
    TcParams tp;
    tp.R = static_cast<float*>(p.R);
    tp.ldr = p.ldr;
    tp.M = M;
    tp.N = N;
    tp.K3 = 3 * K;
    tp.tiles_m = static_cast<int32_t>((M + BM - 1) / BM);
    tp.tiles_n = static_cast<int32_t>((N + BN - 1) / BN);
    tp.group_m = 8;
    tp.r_vec_ok = p.r_vec_ok;
    const int64_t tiles = int64_t(tp.tiles_m) * tp.tiles_n;
    tf32x3_gemm_kernel<Cfg><<<static_cast<unsigned>(tiles), THREADS, Cfg::SMEM, s>>>(ma, mb, tp);
    return cudaGetLastError();
}

cudaError_t no_tile_launch(const KParams&, const CUtensorMap&, const CUtensorMap&, dim3, cudaStream_t) {
    return cudaErrorNotSupported;  // launched through VariantDesc::run
}

}  // namespace tc

template <class Cfg>
void add_tc(Registry& reg, const char* name) {
    VariantDesc v;
    v.body = 0;   // AMLT_BODY_GEMM
    v.dtype = 1;  // AMLT_F32
    v.bm = tc::BM;
    v.bn = Cfg::BN;
    v.bk = tc::BK;
    v.tm = tc::BM;
    v.tn = Cfg::BN;
    v.threads = tc::THREADS;
    v.stages = Cfg::STAGES;
    v.smem = Cfg::SMEM;
    v.minb = 1;
    v.vec = true;
    v.tc = true;
    v.name = name;
    v.func = reinterpret_cast<const void*>(&tc::tf32x3_gemm_kernel<Cfg>);
    v.launch = &tc::no_tile_launch;
    v.ws_bytes = &tc::ws_bytes;
    v.run = &tc::run<Cfg>;
    v.prep_b = &tc::prep_b;
    v.prep_id = 1;  // 3xTF32 split of B, shared by both tile shapes
    reg.variants.push_back(v);
}

void register_tcgen05_gemm(Registry& reg) {
    add_tc<tc::Wide>(reg, "tcgen05_3xtf32");
    add_tc<tc::Narrow>(reg, "tcgen05_3xtf32_acc4");
}

}  // namespace amltk
