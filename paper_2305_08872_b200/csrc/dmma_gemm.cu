// dmma_gemm.cu — plain-GEMM body in fp64 on the FP64 tensor cores.
//
//   R[i][j] += sum_k A[i][k] * B[k][j]        (preset matmul, presets.cpp:64-65)
//
// tcgen05.mma has no f64 kind (its kinds are f16, tf32, f8f6f4, i8, mx*), so
// the sm_100a fp64 tensor path is the warp-level `mma.sync.m8n8k4.f64`,
// which lowers to DMMA. Everything else follows the CUDA-core kernels: a
// STAGES-deep cp.async ring stages A (BM x BK) and B (BK x BN) tiles, with
// row padding chosen so the fragment loads are bank-conflict free:
//   A fragment  lane -> As[m + lane/4][k + lane%4]   (row stride BK+4 doubles)
//   B fragment  lane -> Bs[k + lane%4][n + lane/4]   (row stride BN+4 doubles)
// Each warp owns a (WTM*8) x (WTN*8) accumulator tile in registers.
#include "variants.h"

namespace amltk {

__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
    asm volatile(
        "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
        : "+d"(d[0]), "+d"(d[1])
        : "d"(a), "d"(b));
}

template <int WTM, int WTN, int WARPS_M, int WARPS_N, int BK, int STAGES>
struct DmmaCfg {
    static constexpr int THREADS = 32 * WARPS_M * WARPS_N;
    static constexpr int BM = WTM * 8 * WARPS_M;
    static constexpr int BN = WTN * 8 * WARPS_N;
    static constexpr int LDA_S = BK + 4;  // padded smem row strides (doubles)
    static constexpr int LDB_S = BN + 4;
    static constexpr int SMEM_A = BM * LDA_S;
    static constexpr int SMEM_B = BK * LDB_S;
    static constexpr int SMEM_BYTES = STAGES * (SMEM_A + SMEM_B) * 8;
};

template <int WTM, int WTN, int WARPS_M, int WARPS_N, int BK, int STAGES, int MINB>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N, MINB) dmma_gemm_kernel(const KParams p) {
    using Cfg = DmmaCfg<WTM, WTN, WARPS_M, WARPS_N, BK, STAGES>;
    constexpr int THREADS = Cfg::THREADS;
    constexpr int BM = Cfg::BM, BN = Cfg::BN;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double* As = reinterpret_cast<double*>(smem_raw);
    double* Bs = As + STAGES * Cfg::SMEM_A;

    const int G = p.group_m;
    const int bid = blockIdx.x;
    const int per_group = G * p.tiles_n;
    const int group = bid / per_group;
    const int first_m = group * G;
    const int gsize = min(p.tiles_m - first_m, G);
    const int in_group = bid - group * per_group;
    const int64_t m0 = static_cast<int64_t>(first_m + in_group % gsize) * BM;
    const int64_t n0 = static_cast<int64_t>(in_group / gsize) * BN;
    const int split = blockIdx.y;
    const int64_t kbeg = static_cast<int64_t>(split) * p.kslice;
    const int64_t kspan = min(p.kslice, p.K - kbeg);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WARPS_N, wn = warp - wm * WARPS_N;
    const double* __restrict__ Ag = static_cast<const double*>(p.A);
    const double* __restrict__ Bg = static_cast<const double*>(p.B);

    auto load_tile = [&](int stage, int64_t k0) {
        double* as = As + stage * Cfg::SMEM_A;
        double* bs = Bs + stage * Cfg::SMEM_B;
        const int64_t kend = kbeg + kspan;
        constexpr int ACH = BK / 2;
        for (int c = tid; c < BM * ACH; c += THREADS) {
            const int row = c / ACH, kc = (c - row * ACH) * 2;
            const int64_t gi = m0 + row, gk = k0 + kc;
            int64_t rem = gi < p.M ? kend - gk : 0;
            rem = rem < 0 ? 0 : (rem > 2 ? 2 : rem);
            cp_async16(as + row * Cfg::LDA_S + kc, rem > 0 ? Ag + gi * p.lda + gk : Ag,
                       static_cast<int>(rem * 8));
        }
        constexpr int BCH = BN / 2;
        for (int c = tid; c < BK * BCH; c += THREADS) {
            const int kr = c / BCH, cc = (c - kr * BCH) * 2;
            const int64_t gk = k0 + kr, gj = n0 + cc;
            int64_t rem = gk < kend ? p.N - gj : 0;
            rem = rem < 0 ? 0 : (rem > 2 ? 2 : rem);
            cp_async16(bs + kr * Cfg::LDB_S + cc, rem > 0 ? Bg + gk * p.ldb + gj : Bg,
                       static_cast<int>(rem * 8));
        }
    };

    double acc[WTM][WTN][2];
#pragma unroll
    for (int a = 0; a < WTM; ++a)
#pragma unroll
        for (int b = 0; b < WTN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    const int nkt = static_cast<int>((kspan + BK - 1) / BK);
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < nkt) load_tile(s, kbeg + static_cast<int64_t>(s) * BK);
        cp_async_commit();
    }
    const int fr = lane >> 2, fk = lane & 3;
    for (int kt = 0; kt < nkt; ++kt) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nxt = kt + STAGES - 1;
            if (nxt < nkt) load_tile(nxt % STAGES, kbeg + static_cast<int64_t>(nxt) * BK);
            cp_async_commit();
        }
        const int stage = kt % STAGES;
        const double* as = As + stage * Cfg::SMEM_A + (wm * WTM * 8 + fr) * Cfg::LDA_S + fk;
        const double* bs = Bs + stage * Cfg::SMEM_B + fk * Cfg::LDB_S + wn * WTN * 8 + fr;
        // zero-filled k positions (past k1) multiply 0 * 0: no contribution
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[WTM], bf[WTN];
#pragma unroll
            for (int a = 0; a < WTM; ++a) af[a] = as[a * 8 * Cfg::LDA_S + kk];
#pragma unroll
            for (int b = 0; b < WTN; ++b) bf[b] = bs[kk * Cfg::LDB_S + b * 8];
#pragma unroll
            for (int a = 0; a < WTM; ++a)
#pragma unroll
                for (int b = 0; b < WTN; ++b) dmma_884(acc[a][b], af[a], bf[b]);
        }
    }
    cp_async_wait<0>();

    // C fragment: lane holds C[lane/4][2*(lane%4) + {0,1}]
    double* Rg = static_cast<double*>(p.R);
    double* Wg = static_cast<double*>(p.work);
#pragma unroll
    for (int a = 0; a < WTM; ++a) {
        const int64_t gi = m0 + wm * WTM * 8 + a * 8 + fr;
        if (gi >= p.M) continue;
#pragma unroll
        for (int b = 0; b < WTN; ++b) {
            const int64_t gj = n0 + wn * WTN * 8 + b * 8 + 2 * fk;
            if (p.splits > 1) {
                double* dst = Wg + (static_cast<int64_t>(split) * p.M + gi) * p.N + gj;
                if (gj < p.N) dst[0] = acc[a][b][0];
                if (gj + 1 < p.N) dst[1] = acc[a][b][1];
            } else {
                double* dst = Rg + gi * p.ldr + gj;
                if (p.r_vec_ok && gj + 2 <= p.N) {
                    double2 o = p.r_zero ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(dst);
                    o.x += acc[a][b][0];
                    o.y += acc[a][b][1];
                    *reinterpret_cast<double2*>(dst) = o;
                } else {
                    if (gj < p.N) dst[0] = (p.r_zero ? 0.0 : dst[0]) + acc[a][b][0];
                    if (gj + 1 < p.N) dst[1] = (p.r_zero ? 0.0 : dst[1]) + acc[a][b][1];
                }
            }
        }
    }
}

template <int WTM, int WTN, int WARPS_M, int WARPS_N, int BK, int STAGES, int MINB>
cudaError_t launch_dmma(const KParams& p, const CUtensorMap&, const CUtensorMap&, dim3 grid,
                        cudaStream_t s) {
    using Cfg = DmmaCfg<WTM, WTN, WARPS_M, WARPS_N, BK, STAGES>;
    dmma_gemm_kernel<WTM, WTN, WARPS_M, WARPS_N, BK, STAGES, MINB>
        <<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(p);
    return cudaGetLastError();
}

template <int WTM, int WTN, int WARPS_M, int WARPS_N, int BK, int STAGES, int MINB>
void add_dmma(Registry& reg, const char* name) {
    using Cfg = DmmaCfg<WTM, WTN, WARPS_M, WARPS_N, BK, STAGES>;
    VariantDesc v;
    v.body = 0;   // AMLT_BODY_GEMM
    v.dtype = 0;  // AMLT_F64
    v.bm = Cfg::BM;
    v.bn = Cfg::BN;
    v.bk = BK;
    v.tm = WTM * 8;
    v.tn = WTN * 8;
    v.threads = Cfg::THREADS;
    v.stages = STAGES;
    v.smem = Cfg::SMEM_BYTES;
    v.minb = MINB;
    v.vec = true;
    v.tc = true;
    v.r_overwrite = true;
    v.name = name;
    v.func = reinterpret_cast<const void*>(&dmma_gemm_kernel<WTM, WTN, WARPS_M, WARPS_N, BK, STAGES, MINB>);
    v.launch = &launch_dmma<WTM, WTN, WARPS_M, WARPS_N, BK, STAGES, MINB>;
    reg.variants.push_back(v);
}

void register_dmma_gemm(Registry& reg) {
    //       WTM WTN WM WN BK ST MINB
    add_dmma<8, 4, 2, 4, 16, 3, 1>(reg, "dmma_w64x32_c2x4");
    add_dmma<4, 4, 2, 4, 16, 3, 2>(reg, "dmma_w32x32_c2x4");
    add_dmma<4, 4, 2, 2, 16, 4, 3>(reg, "dmma_w32x32_c2x2");
}

}  // namespace amltk
