// mixbench.cu — throughput of fp64 instruction mixes on one SM (scratch
// experiment, not product code). Each thread runs NCH independent chains;
// grid = SMs x BLK blocks of 256 threads. Prints cycles per warp-iteration per
// SMSP for each mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mixbench tools/mixbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int NCH = 16;
constexpr int ITERS = 2048;

template <int MIX>
__global__ void __launch_bounds__(256) mix(double* out, const double* in, int n) {
    double a[NCH], b[NCH], acc[NCH];
    const double t = in[0], c1 = in[1];
    double tt[4], cc[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        tt[c] = in[18 + (threadIdx.x + c) % 8];
        cc[c] = in[26 + c % 4];
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        a[c] = in[2 + (threadIdx.x + c) % 8];
        b[c] = in[10 + (threadIdx.x * 3 + c) % 8];
        acc[c] = 0;
    }
    __shared__ __align__(16) double sA[16 * 8 * 4];
    __shared__ __align__(16) double sB[16 * 128];
    if constexpr (MIX == 8) {
        for (int i = threadIdx.x; i < 16 * 8 * 4; i += blockDim.x) sA[i] = in[i % 16];
        for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) sB[i] = in[(i * 7) % 16];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if constexpr (MIX >= 22 && MIX <= 27) {
        // theta form of discount: per (k, j) a threshold theta on a and the
        // two candidate b values; P = a > theta; acc = fma(a, P ? x1 : x0, acc).
        // 22: 4x4 tile, registers; 23: 4x4 tile from smem; 24: 8x4 from smem;
        // 25: original discount 8x4 from smem (reference point for 24)
        constexpr int RR = (MIX == 24 || MIX == 25 || MIX == 26 || MIX == 27) ? 8 : 4;
        double th[4], x0[4], x1[4], aa[8], acc2[RR * 4];
#pragma unroll
        for (int c = 0; c < 4; ++c) { th[c] = in[18 + c]; x0[c] = in[22 + c]; x1[c] = in[26 + c]; }
#pragma unroll
        for (int c = 0; c < RR * 4; ++c) acc2[c] = 0;
        __shared__ __align__(16) double sT[8 * 128 * 3];
        for (int i = threadIdx.x; i < 8 * 128 * 3; i += blockDim.x) sT[i] = in[(i * 7) % 32];
        for (int i = threadIdx.x; i < 16 * 8 * 4; i += blockDim.x) sA[i] = in[i % 16];
        __syncthreads();
        for (int it = 0; it < n; ++it) {
            const int k = it & 7;
            if constexpr (MIX == 22) {
#pragma unroll
                for (int c = 0; c < 4; ++c) { asm volatile("" : "+d"(th[c]), "+d"(x0[c]), "+d"(x1[c])); }
#pragma unroll
                for (int r = 0; r < 4; ++r) { aa[r] = a[r]; asm volatile("" : "+d"(aa[r])); }
            } else {
                const double* row = sT + k * 384;
                const double2 t01 = *reinterpret_cast<const double2*>(row + lane * 2);
                const double2 t23 = *reinterpret_cast<const double2*>(row + 64 + lane * 2);
                const double2 p01 = *reinterpret_cast<const double2*>(row + 128 + lane * 2);
                const double2 p23 = *reinterpret_cast<const double2*>(row + 192 + lane * 2);
                const double2 q01 = *reinterpret_cast<const double2*>(row + 256 + lane * 2);
                const double2 q23 = *reinterpret_cast<const double2*>(row + 320 + lane * 2);
                th[0] = t01.x; th[1] = t01.y; th[2] = t23.x; th[3] = t23.y;
                x0[0] = p01.x; x0[1] = p01.y; x0[2] = p23.x; x0[3] = p23.y;
                x1[0] = q01.x; x1[1] = q01.y; x1[2] = q23.x; x1[3] = q23.y;
#pragma unroll
                for (int r = 0; r < RR; ++r) aa[r] = sA[(warp * 8 + r) % 32 * 16 + k];
            }
#pragma unroll
            for (int c = 0; c < RR * 4; ++c) {
                if constexpr (MIX == 26) {  // predicated DFMA pair, no select
                    asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; @P fma.rn.f64 %0, %1, %3, %0; "
                        "@!P fma.rn.f64 %0, %1, %4, %0; }"
                        : "+d"(acc2[c]) : "d"(aa[c / 4]), "d"(th[c % 4]), "d"(x1[c % 4]), "d"(x0[c % 4]));
                } else if constexpr (MIX == 27) {  // theta form via selp.f64
                    asm("{ .reg .pred P; .reg .f64 s; setp.gt.f64 P, %1, %2; selp.f64 s, %3, %4, P; "
                        "fma.rn.f64 %0, %1, s, %0; }"
                        : "+d"(acc2[c]) : "d"(aa[c / 4]), "d"(th[c % 4]), "d"(x1[c % 4]), "d"(x0[c % 4]));
                } else if constexpr (MIX == 25) {
                    double p = __dmul_rn(aa[c / 4], x0[c % 4]);
                    double f = p > th[c % 4] ? x1[c % 4] : 1.0;
                    acc2[c] = __fma_rn(p, f, acc2[c]);
                } else {
                    double bs = aa[c / 4] > th[c % 4] ? x1[c % 4] : x0[c % 4];
                    acc2[c] = __fma_rn(aa[c / 4], bs, acc2[c]);
                }
            }
        }
        double s = 0;
#pragma unroll
        for (int c = 0; c < RR * 4; ++c) s += acc2[c];
        if (s == 1234.5) out[threadIdx.x] = s;
        return;
    }
    if constexpr (MIX == 11 || MIX == 12) {
        // B only from smem, A in registers. MIX 11: 4 x LDS.64 per k (one per
        // column); MIX 12: column-major B tile, one LDS.128 = 2 k values of a
        // column, 4 per 2 k.
        for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) sB[i] = in[(i * 7) % 16];
        __syncthreads();
        for (int it = 0; it < n; it += 4) {
#pragma unroll
            for (int kk = 0; kk < 4; kk += 2) {
                const int k = (it + kk) & 15;
                double bb[2][4];
                if constexpr (MIX == 11) {
#pragma unroll
                    for (int v = 0; v < 2; ++v)
#pragma unroll
                        for (int c = 0; c < 4; ++c) bb[v][c] = sB[(k + v) * 128 + c * 32 + lane];
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const double2 t2 = *reinterpret_cast<const double2*>(
                            sB + ((c * 32 + lane) * 16 + k) % (16 * 128));
                        bb[0][c] = t2.x;
                        bb[1][c] = t2.y;
                    }
                }
#pragma unroll
                for (int v = 0; v < 2; ++v)
#pragma unroll
                    for (int c = 0; c < NCH; ++c) {
                        double p = __dmul_rn(a[c / 4], bb[v][c % 4]);
                        double f = p > tt[c % 4] ? cc[c % 4] : 1.0;
                        acc[c] = __fma_rn(p, f, acc[c]);
                    }
            }
        }
    } else
    if constexpr (MIX == 9 || MIX == 10) {
        // MIX 9: 4x4 tile fed from smem, 4 k per loop trip (loads hoistable);
        // MIX 10: same with only the B loads (A from registers)
        for (int i = threadIdx.x; i < 16 * 8 * 4; i += blockDim.x) sA[i] = in[i % 16];
        for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) sB[i] = in[(i * 7) % 16];
        __syncthreads();
        for (int it = 0; it < n; it += 4) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int k = (it + kk) & 15;
                const double2 b01 = *reinterpret_cast<const double2*>(sB + k * 128 + lane * 2);
                const double2 b23 = *reinterpret_cast<const double2*>(sB + k * 128 + 64 + lane * 2);
                double bb[4] = {b01.x, b01.y, b23.x, b23.y};
                double aa[4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    aa[r] = MIX == 9 ? sA[(warp * 4 + r) * 16 + k] : a[r];
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    double p = __dmul_rn(aa[c / 4], bb[c % 4]);
                    double f = p > tt[c % 4] ? cc[c % 4] : 1.0;
                    acc[c] = __fma_rn(p, f, acc[c]);
                }
            }
        }
    } else
    for (int it = 0; it < n; ++it) {
        if constexpr (MIX == 8) {
            // the tiled kernel's operand traffic: per k, B = 4 lane-interleaved
            // columns (2 x LDS.128), A = 4 rows broadcast (LDS.64 each)
            const int k = it & 15;
            const double2 b01 = *reinterpret_cast<const double2*>(sB + k * 128 + lane * 2);
            const double2 b23 = *reinterpret_cast<const double2*>(sB + k * 128 + 64 + lane * 2);
            b[0] = b01.x; b[1] = b01.y; b[2] = b23.x; b[3] = b23.y;
#pragma unroll
            for (int r = 0; r < 4; ++r) a[r] = sA[(warp * 4 + r) * 16 + k];
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            if constexpr (MIX == 8) {
                double p = __dmul_rn(a[c / 4], b[c % 4]);
                double f = p > tt[c % 4] ? cc[c % 4] : 1.0;
                acc[c] = __fma_rn(p, f, acc[c]);
            }
            if constexpr (MIX == 0) {  // DFMA, three distinct fresh sources
                acc[c] = __fma_rn(a[c], b[c], acc[c]);
            } else if constexpr (MIX == 1) {  // discount: DMUL DSETP 2xFSEL DFMA
                double p = __dmul_rn(a[c], b[c]);
                double f = p > t ? c1 : 1.0;
                acc[c] = __fma_rn(p, f, acc[c]);
            } else if constexpr (MIX == 2) {  // DMUL + DFMA(p, c1, acc)
                double p = __dmul_rn(a[c], b[c]);
                acc[c] = __fma_rn(p, c1, acc[c]);
            } else if constexpr (MIX == 3) {  // DMUL + DSETP + DADD predicated-select
                double p = __dmul_rn(a[c], b[c]);
                acc[c] = p > t ? acc[c] + p : acc[c];
            } else if constexpr (MIX == 4) {  // DFMA sharing a (reuse slot)
                acc[c] = __fma_rn(a[0], b[c], acc[c]);
            } else if constexpr (MIX == 5) {  // discount, select p instead: 2 accs
                double p = __dmul_rn(a[c], b[c]);
                acc[c] = __dadd_rn(acc[c], p > t ? p * c1 : p);
            } else if constexpr (MIX == 6) {  // discount with per-column t, c1 (4 columns)
                double p = __dmul_rn(a[c], b[c]);
                double f = p > tt[c % 4] ? cc[c % 4] : 1.0;
                acc[c] = __fma_rn(p, f, acc[c]);
            } else if constexpr (MIX == 13) {  // DMUL chains only
                acc[c] = __dmul_rn(acc[c], b[c]);
            } else if constexpr (MIX == 14) {  // DADD chains only
                acc[c] = __dadd_rn(acc[c], b[c]);
            } else if constexpr (MIX == 15) {  // DSETP + 2 FSEL only (acc = select)
                acc[c] = b[c] > acc[c] ? c1 : 1.0;
            } else if constexpr (MIX == 16) {  // DMUL, DSETP, 1 SEL (hi word) -> m, DFMA c, DFMA acc
                double p = __dmul_rn(a[c], b[c]);
                unsigned hi;
                asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; selp.b32 %0, 0x3ff00000, 0, P; }"
                    : "=r"(hi) : "d"(p), "d"(t));
                double m = __hiloint2double(int(hi), 0);
                double cf = __fma_rn(-m, c1, 1.0);
                acc[c] = __fma_rn(p, cf, acc[c]);
            } else if constexpr (MIX == 17) {  // predicated DFMA / DADD
                double p = __dmul_rn(a[c], b[c]);
                asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; @P fma.rn.f64 %0, %1, %3, %0; "
                    "@!P add.rn.f64 %0, %0, %1; }" : "+d"(acc[c]) : "d"(p), "d"(t), "d"(c1));
            } else if constexpr (MIX == 18) {  // two accumulators: DFMA all, @P DADD masked
                double p = __dmul_rn(a[c], b[c]);
                asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; @P add.rn.f64 %0, %0, %1; }"
                    : "+d"(a[(c + 1) % NCH]) : "d"(p), "d"(t));
                acc[c] = __dadd_rn(acc[c], p);
            } else if constexpr (MIX == 19) {  // DSETP + DADD (pred add)
                asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; @P add.rn.f64 %0, %0, %1; }"
                    : "+d"(acc[c]) : "d"(b[c]), "d"(t));
            } else if constexpr (MIX == 20) {  // DMUL + DSETP + 1 SEL only
                double p = __dmul_rn(a[c], b[c]);
                unsigned hi;
                asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; selp.b32 %0, 0x3ff00000, 0, P; }"
                    : "=r"(hi) : "d"(p), "d"(t));
                acc[c] = __hiloint2double(int(hi) ^ __double2hiint(acc[c]), 0);
            } else if constexpr (MIX == 21) {  // DSETP alone (predicate feeds an int add)
                unsigned hi;
                asm("{ .reg .pred P; setp.gt.f64 P, %1, %2; selp.b32 %0, 1, 0, P; }"
                    : "=r"(hi) : "d"(b[c]), "d"(acc[c]));
                acc[c] = __hiloint2double(__double2hiint(acc[c]) + int(hi), __double2loint(acc[c]));
            } else if constexpr (MIX == 7) {  // discount, 4x4 tile: a per row, b/t/c1 per col
                double p = __dmul_rn(a[c / 4], b[c % 4]);
                double f = p > tt[c % 4] ? cc[c % 4] : 1.0;
                acc[c] = __fma_rn(p, f, acc[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) asm volatile("" : "+d"(b[c]));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) s += acc[c];
    if (s == 1234.5) out[threadIdx.x] = s;
}

template <int MIX>
void run(int sms, int blk, const char* name, double* out, const double* in) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    mix<MIX><<<sms * blk, 256>>>(out, in, ITERS);
    cudaEventRecord(e0);
    mix<MIX><<<sms * blk, 256>>>(out, in, ITERS);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int nch = (MIX == 24 || MIX == 25 || MIX == 26 || MIX == 27) ? 32 : NCH;
    double warp_iters_per_smsp = double(blk) * 8 * nch * ITERS / 4.0;
    double cycles = ms * 1e-3 * clk * 1e3;  // at max clock
    printf("%-44s blk=%d  %.3f ms  %.2f cycles/warp-iter/SMSP (at max clock)\n", name, blk, ms,
           cycles / warp_iters_per_smsp);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out, *in;
    cudaMalloc(&out, 1024 * 8);
    cudaMalloc(&in, 64 * 8);
    double h[64];
    for (int i = 0; i < 64; ++i) h[i] = 1.0 + i * 0.25;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int blk : {1, 2}) {
        run<7>(sms, blk, "discount 4x4 tile regs (reference point)", out, in);
        run<22>(sms, blk, "theta form 4x4 regs: DSETP 2SEL DFMA", out, in);
        run<8>(sms, blk, "discount 4x4 tile smem (reference point)", out, in);
        run<23>(sms, blk, "theta form 4x4 smem (3 planes)", out, in);
        run<25>(sms, blk, "discount 8x4 smem (reference point)", out, in);
        run<24>(sms, blk, "theta form 8x4 smem (3 planes)", out, in);
        run<26>(sms, blk, "theta 8x4 smem, predicated DFMA pair", out, in);
        run<27>(sms, blk, "theta 8x4 smem, selp.f64", out, in);
    }
    if (getenv("MIX_ALL") == nullptr) return 0;
    for (int blk : {2, 4}) {
        run<13>(sms, blk, "DMUL only", out, in);
        run<14>(sms, blk, "DADD only", out, in);
        run<15>(sms, blk, "DSETP + 2 FSEL only", out, in);
        run<16>(sms, blk, "discount via m: DMUL DSETP SEL DFMA DFMA", out, in);
        run<17>(sms, blk, "discount predicated @P DFMA / @!P DADD", out, in);
        run<18>(sms, blk, "two accs: DMUL DSETP @P DADD DADD", out, in);
        run<19>(sms, blk, "DSETP + @P DADD", out, in);
        run<20>(sms, blk, "DMUL DSETP SEL (+int ops)", out, in);
        run<21>(sms, blk, "DSETP SEL IADD", out, in);
    }
    for (int blk : {1, 2, 4}) {
        run<0>(sms, blk, "DFMA a,b,acc (3 fresh)", out, in);
        run<4>(sms, blk, "DFMA a0(shared),b,acc", out, in);
        run<1>(sms, blk, "discount DMUL DSETP 2FSEL DFMA", out, in);
        run<2>(sms, blk, "DMUL + DFMA(p,c1,acc)", out, in);
        run<3>(sms, blk, "DMUL DSETP DADD-select", out, in);
        run<5>(sms, blk, "DMUL DSETP DMUL-select DADD", out, in);
        run<6>(sms, blk, "discount, per-column t/c1 (4 cols)", out, in);
        run<7>(sms, blk, "discount 4x4 tile (a per row, b/t/c1 per col)", out, in);
        run<8>(sms, blk, "discount 4x4 tile, operands from smem", out, in);
        run<9>(sms, blk, "discount 4x4, smem, 4 k unrolled", out, in);
        run<10>(sms, blk, "discount 4x4, smem B only, 4 k unrolled", out, in);
        run<11>(sms, blk, "discount 4x4, smem B only, LDS.64 per column", out, in);
        run<12>(sms, blk, "discount 4x4, smem B only, col-major LDS.128 (2 k)", out, in);
    }
    return 0;
}
