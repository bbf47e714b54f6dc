// thetabench.cu — throughput of forms of the theta-discount step (scratch
// experiment, not product code). 8 x 4 micro-tile per thread: a[8] per row,
// (theta, x0, x1)[4] per column. FORMs 0-7 keep the operands in registers
// behind empty asm statements; ptxas does not see those, so it hoists the
// compare and selects out of the loop and they time the DFMA alone (not
// run). FORMs 8-17 load the operands from shared memory every k, as the tile
// kernel does. Prints cycles per
// warp-product per SMSP at the measured clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o thetabench tools/thetabench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

constexpr int TM = 8, TN = 4, ITERS = 4096;

__device__ __forceinline__ unsigned hi(double x) { return static_cast<unsigned>(__double2hiint(x)); }
__device__ __forceinline__ unsigned lo(double x) { return static_cast<unsigned>(__double2loint(x)); }

template <int FORM>
__global__ void __launch_bounds__(384, 1) kern(double* out, const double* in, long long* cyc) {
    double a[TM], th[TN], x0[TN], x1[TN], acc[TM][TN];
    double acc2[TM][TN] = {};
    int cnt[TM][TN] = {};
    float ahf[TM], thf[TN];
    const int t = threadIdx.x;
#pragma unroll
    for (int r = 0; r < TM; ++r) a[r] = in[(t + r) & 63];
#pragma unroll
    for (int c = 0; c < TN; ++c) {
        th[c] = in[64 + ((t + 3 * c) & 63)];
        x0[c] = in[128 + ((t + 5 * c) & 63)];
        x1[c] = in[192 + ((t + 7 * c) & 63)];
    }
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[r][c] = 0.0;
    // shared tiles for the smem-fed forms: A as [rows][16 k] (row-broadcast
    // reads, as the tile kernel), B planes as [3][8 k][128 cols]
    __shared__ __align__(16) double sA[96 * 16];
    __shared__ __align__(16) double sB[3 * 8 * 128];
    __shared__ __align__(16) unsigned sAh[96 * 16];  // (a, a) as f16x2
    __shared__ __align__(16) __half2 sTh[8 * 128];
    for (int i = t; i < 96 * 16; i += blockDim.x) sA[i] = in[i & 63];
    for (int i = t; i < 3 * 8 * 128; i += blockDim.x) sB[i] = in[64 + (i & 191)];
    for (int i = t; i < 96 * 16; i += blockDim.x) sAh[i] = __half_as_ushort(__double2half(in[i & 63])) * 0x10001u;
    for (int i = t; i < 8 * 128; i += blockDim.x) sTh[i] = __halves2half2(__double2half(in[64 + (i & 63)]), __double2half(in[64 + ((i + 1) & 63)]));
    __syncthreads();
    const int lane = t & 31, warp = t >> 5;
    // runtime 2 and -1 (in[0] is 0): keeps ptxas from strength-reducing the
    // IMAD-based forms into shifts and adds on the ALU
    const unsigned k2 = static_cast<unsigned>(in[0] + 2.0);
    const int kneg = -static_cast<int>(in[0] + 1.0);
    const long long c0 = clock64();
    if constexpr (FORM >= 8) {
        // smem-fed: 8: row outer, loads then compute per k; 9: loads for the next
        // k issued before this k's compute (register double buffer); 10: B from
        // smem, a from registers; 11: a from smem, B from registers
        double na[TM], nth[TN], nx0[TN], nx1[TN];
        unsigned la16[TM], lt16[TN / 2];
        auto load = [&](int k, double* la, double* lth, double* lx0, double* lx1) {
            if constexpr (FORM != 10) {
#pragma unroll
                for (int r = 0; r < TM; ++r) la[r] = sA[(warp * 8 + r) * 16 + k];
            }
            if constexpr (FORM == 22 || FORM == 23) {
#pragma unroll
                for (int r = 0; r < TM; ++r) la16[r] = sAh[(warp * 8 + r) * 16 + k];
#pragma unroll
                for (int q = 0; q < TN / 2; ++q) lt16[q] = *reinterpret_cast<const unsigned*>(&sTh[k * 128 + q * 64 + lane]);
            }
            if constexpr (FORM != 11) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    const double2 t2 = *reinterpret_cast<const double2*>(sB + k * 128 + q * 64 + lane * 2);
                    const double2 p2 = *reinterpret_cast<const double2*>(sB + 1024 + k * 128 + q * 64 + lane * 2);
                    const double2 x2 = *reinterpret_cast<const double2*>(sB + 2048 + k * 128 + q * 64 + lane * 2);
                    lth[2 * q] = t2.x; lth[2 * q + 1] = t2.y;
                    lx0[2 * q] = p2.x; lx0[2 * q + 1] = p2.y;
                    lx1[2 * q] = x2.x; lx1[2 * q + 1] = x2.y;
                }
            }
        };
        auto compute = [&](const double* la, const double* lth, const double* lx0, const double* lx1) {
            if constexpr (FORM == 13 || FORM == 14) {  // compare the high words (f32 / s32)
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        bool m;
                        if constexpr (FORM == 13)
                            m = __uint_as_float(hi(la[r])) > __uint_as_float(hi(lth[c]));
                        else
                            m = static_cast<int>(hi(la[r])) > static_cast<int>(hi(lth[c]));
                        acc[r][c] = __fma_rn(la[r], m ? lx1[c] : lx0[c], acc[r][c]);
                    }
                return;
            }
            if constexpr (FORM == 22 || FORM == 23) {  // fp16x2 compare (HSETP2, 2 masks per instruction) + 2 FSEL + DFMA
#pragma unroll
                for (int q = 0; q < TN / 2; ++q) {
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        const unsigned a2 = la16[r], th2 = lt16[q];
                        if constexpr (FORM == 22)
                            asm("{\n .reg .pred p, q;\n .reg .b32 l0, h0, l1, h1, x0l, x0h, x1l, x1h, y0l, y0h, y1l, y1h;\n"
                                " .reg .f64 x0, x1;\n"
                                " setp.gt.f16x2 p|q, %2, %3;\n"
                                " mov.b64 {x0l, x0h}, %5; mov.b64 {x1l, x1h}, %6; mov.b64 {y0l, y0h}, %7; mov.b64 {y1l, y1h}, %8;\n"
                                " selp.b32 l0, y0l, x0l, p; selp.b32 h0, y0h, x0h, p;\n"
                                " selp.b32 l1, y1l, x1l, q; selp.b32 h1, y1h, x1h, q;\n"
                                " mov.b64 x0, {l0, h0}; mov.b64 x1, {l1, h1};\n"
                                " fma.rn.f64 %0, %4, x0, %0; fma.rn.f64 %1, %4, x1, %1;\n}\n"
                                : "+d"(acc[r][2 * q]), "+d"(acc[r][2 * q + 1])
                                : "r"(a2), "r"(th2), "d"(la[r]), "d"(lx0[2 * q]), "d"(lx0[2 * q + 1]), "d"(lx1[2 * q]),
                                  "d"(lx1[2 * q + 1]));
                        else
                            asm("{\n .reg .pred p, q;\n .reg .b32 l0, h0, l1, h1, x0l, x0h, x1l, x1h, y0l, y0h, y1l, y1h;\n"
                                " setp.gt.f16x2 p|q, %2, %3;\n"
                                " mov.b64 {x0l, x0h}, %0; mov.b64 {x1l, x1h}, %1; mov.b64 {y0l, y0h}, %4; mov.b64 {y1l, y1h}, %5;\n"
                                " selp.b32 l0, y0l, x0l, p; selp.b32 h0, y0h, x0h, p;\n"
                                " selp.b32 l1, y1l, x1l, q; selp.b32 h1, y1h, x1h, q;\n"
                                " mov.b64 %0, {l0, h0}; mov.b64 %1, {l1, h1};\n}\n"
                                : "+d"(acc[r][2 * q]), "+d"(acc[r][2 * q + 1])
                                : "r"(a2), "r"(th2), "d"(lx1[2 * q]), "d"(lx1[2 * q + 1]));
                    }
                }
                return;
            }
            if constexpr (FORM == 24) {  // ISETP (high words) + SEL hi(a) + 2 DFMA: acc += a*x0 + (m ? a : 0)*d
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        const int h = __double2hiint(la[r]);
                        const double y = __hiloint2double(h > __double2hiint(lth[c]) ? h : 0, 0);
                        acc[r][c] = __fma_rn(y, lx1[c], __fma_rn(la[r], lx0[c], acc[r][c]));
                    }
                return;
            }
            if constexpr (FORM == 25) {  // theta form as one PTX block per column: 8 DSETP, 8+8 SELP, 8 DFMA
#pragma unroll
                for (int c = 0; c < TN; ++c) {
                    asm("{\n .reg .pred p<8>; .reg .b32 l<8>, h<8>; .reg .f64 x<8>;\n"
                        " .reg .b32 x0l, x0h, x1l, x1h;\n"
                        " mov.b64 {x0l, x0h}, %9; mov.b64 {x1l, x1h}, %10;\n"
                        " setp.gt.f64 p0, %11, %8; setp.gt.f64 p1, %12, %8; setp.gt.f64 p2, %13, %8; setp.gt.f64 p3, %14, %8;\n"
                        " setp.gt.f64 p4, %15, %8; setp.gt.f64 p5, %16, %8; setp.gt.f64 p6, %17, %8; setp.gt.f64 p7, %18, %8;\n"
                        " selp.b32 l0, x1l, x0l, p0; selp.b32 l1, x1l, x0l, p1; selp.b32 l2, x1l, x0l, p2; selp.b32 l3, x1l, x0l, p3;\n"
                        " selp.b32 l4, x1l, x0l, p4; selp.b32 l5, x1l, x0l, p5; selp.b32 l6, x1l, x0l, p6; selp.b32 l7, x1l, x0l, p7;\n"
                        " selp.b32 h0, x1h, x0h, p0; selp.b32 h1, x1h, x0h, p1; selp.b32 h2, x1h, x0h, p2; selp.b32 h3, x1h, x0h, p3;\n"
                        " selp.b32 h4, x1h, x0h, p4; selp.b32 h5, x1h, x0h, p5; selp.b32 h6, x1h, x0h, p6; selp.b32 h7, x1h, x0h, p7;\n"
                        " mov.b64 x0, {l0, h0}; mov.b64 x1, {l1, h1}; mov.b64 x2, {l2, h2}; mov.b64 x3, {l3, h3};\n"
                        " mov.b64 x4, {l4, h4}; mov.b64 x5, {l5, h5}; mov.b64 x6, {l6, h6}; mov.b64 x7, {l7, h7};\n"
                        " fma.rn.f64 %0, %11, x0, %0; fma.rn.f64 %1, %12, x1, %1; fma.rn.f64 %2, %13, x2, %2; fma.rn.f64 %3, %14, x3, %3;\n"
                        " fma.rn.f64 %4, %15, x4, %4; fma.rn.f64 %5, %16, x5, %5; fma.rn.f64 %6, %17, x6, %6; fma.rn.f64 %7, %18, x7, %7;\n"
                        "}\n"
                        : "+d"(acc[0][c]), "+d"(acc[1][c]), "+d"(acc[2][c]), "+d"(acc[3][c]), "+d"(acc[4][c]),
                          "+d"(acc[5][c]), "+d"(acc[6][c]), "+d"(acc[7][c])
                        : "d"(lth[c]), "d"(lx0[c]), "d"(lx1[c]), "d"(la[0]), "d"(la[1]), "d"(la[2]), "d"(la[3]), "d"(la[4]),
                          "d"(la[5]), "d"(la[6]), "d"(la[7]));
                }
                return;
            }
            if constexpr (FORM == 26) {  // theta form as one PTX block per row: 4 DSETP, 4+4 SELP, 4 DFMA (a reused)
#pragma unroll
                for (int r = 0; r < TM; ++r) {
                    asm("{\n .reg .pred p<4>; .reg .b32 l<4>, h<4>, al<4>, ah<4>, bl<4>, bh<4>; .reg .f64 x<4>;\n"
                        " mov.b64 {al0, ah0}, %9; mov.b64 {al1, ah1}, %10; mov.b64 {al2, ah2}, %11; mov.b64 {al3, ah3}, %12;\n"
                        " mov.b64 {bl0, bh0}, %13; mov.b64 {bl1, bh1}, %14; mov.b64 {bl2, bh2}, %15; mov.b64 {bl3, bh3}, %16;\n"
                        " setp.gt.f64 p0, %4, %5; setp.gt.f64 p1, %4, %6; setp.gt.f64 p2, %4, %7; setp.gt.f64 p3, %4, %8;\n"
                        " selp.b32 l0, bl0, al0, p0; selp.b32 l1, bl1, al1, p1; selp.b32 l2, bl2, al2, p2; selp.b32 l3, bl3, al3, p3;\n"
                        " selp.b32 h0, bh0, ah0, p0; selp.b32 h1, bh1, ah1, p1; selp.b32 h2, bh2, ah2, p2; selp.b32 h3, bh3, ah3, p3;\n"
                        " mov.b64 x0, {l0, h0}; mov.b64 x1, {l1, h1}; mov.b64 x2, {l2, h2}; mov.b64 x3, {l3, h3};\n"
                        " fma.rn.f64 %0, %4, x0, %0; fma.rn.f64 %1, %4, x1, %1; fma.rn.f64 %2, %4, x2, %2; fma.rn.f64 %3, %4, x3, %3;\n"
                        "}\n"
                        : "+d"(acc[r][0]), "+d"(acc[r][1]), "+d"(acc[r][2]), "+d"(acc[r][3])
                        : "d"(la[r]), "d"(lth[0]), "d"(lth[1]), "d"(lth[2]), "d"(lth[3]), "d"(lx0[0]), "d"(lx0[1]),
                          "d"(lx0[2]), "d"(lx0[3]), "d"(lx1[0]), "d"(lx1[1]), "d"(lx1[2]), "d"(lx1[3]));
                }
                return;
            }
            if constexpr (FORM == 18 || FORM == 20) {  // P3: ISETP (high words) + DFMA x0 + predicated DFMA d
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        if constexpr (FORM == 18)
                            asm("{\n .reg .pred p;\n setp.gt.s32 p, %1, %2;\n fma.rn.f64 %0, %3, %4, %0;\n"
                                " @p fma.rn.f64 %0, %3, %5, %0;\n}\n"
                                : "+d"(acc[r][c])
                                : "r"(__double2hiint(la[r])), "r"(__double2hiint(lth[c])), "d"(la[r]), "d"(lx0[c]),
                                  "d"(lx1[c]));
                        else
                            asm("{\n .reg .pred p;\n setp.gt.f64 p, %1, %2;\n fma.rn.f64 %0, %1, %3, %0;\n"
                                " @p fma.rn.f64 %0, %1, %4, %0;\n}\n"
                                : "+d"(acc[r][c])
                                : "d"(la[r]), "d"(lth[c]), "d"(lx0[c]), "d"(lx1[c]));
                    }
                return;
            }
            if constexpr (FORM == 19) {  // P3 grouped per column: 8 ISETP, 8 DFMA x0, 8 predicated DFMA d
#pragma unroll
                for (int c = 0; c < TN; ++c) {
                    asm("{\n .reg .pred p<8>;\n"
                        " setp.gt.s32 p0, %17, %16; setp.gt.s32 p1, %18, %16; setp.gt.s32 p2, %19, %16; setp.gt.s32 p3, %20, %16;\n"
                        " setp.gt.s32 p4, %21, %16; setp.gt.s32 p5, %22, %16; setp.gt.s32 p6, %23, %16; setp.gt.s32 p7, %24, %16;\n"
                        " fma.rn.f64 %0, %8, %25, %0; fma.rn.f64 %1, %9, %25, %1; fma.rn.f64 %2, %10, %25, %2; fma.rn.f64 %3, %11, %25, %3;\n"
                        " fma.rn.f64 %4, %12, %25, %4; fma.rn.f64 %5, %13, %25, %5; fma.rn.f64 %6, %14, %25, %6; fma.rn.f64 %7, %15, %25, %7;\n"
                        " @p0 fma.rn.f64 %0, %8, %26, %0; @p1 fma.rn.f64 %1, %9, %26, %1; @p2 fma.rn.f64 %2, %10, %26, %2; @p3 fma.rn.f64 %3, %11, %26, %3;\n"
                        " @p4 fma.rn.f64 %4, %12, %26, %4; @p5 fma.rn.f64 %5, %13, %26, %5; @p6 fma.rn.f64 %6, %14, %26, %6; @p7 fma.rn.f64 %7, %15, %26, %7;\n"
                        "}\n"
                        : "+d"(acc[0][c]), "+d"(acc[1][c]), "+d"(acc[2][c]), "+d"(acc[3][c]), "+d"(acc[4][c]),
                          "+d"(acc[5][c]), "+d"(acc[6][c]), "+d"(acc[7][c])
                        : "d"(la[0]), "d"(la[1]), "d"(la[2]), "d"(la[3]), "d"(la[4]), "d"(la[5]), "d"(la[6]), "d"(la[7]),
                          "r"(__double2hiint(lth[c])), "r"(__double2hiint(la[0])), "r"(__double2hiint(la[1])),
                          "r"(__double2hiint(la[2])), "r"(__double2hiint(la[3])), "r"(__double2hiint(la[4])),
                          "r"(__double2hiint(la[5])), "r"(__double2hiint(la[6])), "r"(__double2hiint(la[7])),
                          "d"(lx0[c]), "d"(lx1[c]));
                }
                return;
            }
            if constexpr (FORM == 21) {  // 2 DFMA per product, no compare (the P3 FP64 load alone)
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r)
                        acc[r][c] = __fma_rn(la[r], lx1[c], __fma_rn(la[r], lx0[c], acc[r][c]));
                return;
            }
            if constexpr (FORM == 15) {  // DFMA only (the feed plus the FP64 pipe)
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) acc[r][c] = __fma_rn(la[r], lx0[c], acc[r][c]);
                return;
            }
            if constexpr (FORM == 16) {  // DSETP + 2 FSEL only, into the accumulator
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) acc[r][c] = la[r] > lth[c] ? lx1[c] : acc[r][c];
                return;
            }
            if constexpr (FORM == 17) {  // FSETP (high words) + 2 FSEL only, into the accumulator
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r)
                        acc[r][c] = __uint_as_float(hi(la[r])) > __uint_as_float(hi(lth[c])) ? lx1[c] : acc[r][c];
                return;
            }
            if constexpr (FORM >= 27 && FORM <= 30) {
                // exact compare split between the FP64 pipe (DSETP) and the
                // ALU (signed 64-bit compare of the raw bits: exact for a
                // with the sign bit clear): the first NI columns on the ALU
                // (27: 4 of 4, 28: 1 of 4, 29: 2 of 4, 30: 1 of 4 rows-major)
                constexpr int NI = FORM == 27 ? 4 : FORM == 29 ? 2 : 1;
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        bool m;
                        const bool alu = FORM == 30 ? (r % 4 == 0) : (c < NI);
                        if (alu)
                            m = __double_as_longlong(la[r]) > __double_as_longlong(lth[c]);
                        else
                            m = la[r] > lth[c];
                        acc[r][c] = __fma_rn(la[r], m ? lx1[c] : lx0[c], acc[r][c]);
                    }
                return;
            }
            if constexpr (FORM >= 31 && FORM <= 37) {
                // per-column forms (F: DSETP + 2 FSEL; X: ISETP on the high
                // words + 2 FSEL; Y: integer compare of the high words on the
                // FMA pipe, mask by IMAD.HI, select by 2 IMAD; I: DADD
                // theta - a, mask from its sign by IMAD.HI, select by 2 IMAD).
                // Y and X need a >= 0 with zero low words; I is general.
                auto kind = [](int c) {
                    if (FORM == 31) return c == 3 ? 'Y' : 'F';
                    if (FORM == 32) return c == 3 ? 'Y' : c == 2 ? 'X' : 'F';
                    if (FORM == 33) return 'Y';
                    if (FORM == 34) return 'I';
                    if (FORM == 35) return c == 3 ? 'I' : 'F';
                    if (FORM == 36) return c >= 2 ? 'I' : 'F';
                    return c == 3 ? 'Y' : c == 1 ? 'I' : 'F';
                };
#pragma unroll
                for (int c = 0; c < TN; ++c) {
                    const unsigned x0h = hi(lx0[c]), x0l = lo(lx0[c]);
                    const unsigned dh = hi(lx1[c]) - x0h, dl = lo(lx1[c]) - x0l;
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        const char kd = kind(c);
                        if (kd == 'F') {
                            acc[r][c] = __fma_rn(la[r], la[r] > lth[c] ? lx1[c] : lx0[c], acc[r][c]);
                        } else if (kd == 'X') {
                            const bool m = static_cast<int>(hi(la[r])) > static_cast<int>(hi(lth[c]));
                            acc[r][c] = __fma_rn(la[r], m ? lx1[c] : lx0[c], acc[r][c]);
                        } else {
                            unsigned m;
                            if (kd == 'Y') {
                                const int d = static_cast<int>(hi(la[r])) * kneg + static_cast<int>(hi(lth[c]));
                                m = __umulhi(static_cast<unsigned>(d), k2);
                            } else {
                                m = __umulhi(hi(__dsub_rn(lth[c], la[r])), k2);
                            }
                            const double s = __hiloint2double(static_cast<int>(m * dh + x0h), static_cast<int>(m * dl + x0l));
                            acc[r][c] = __fma_rn(la[r], s, acc[r][c]);
                        }
                    }
                }
                return;
            }
            if constexpr (FORM == 38) {
                // boost in theta form: acc += a * (m ? 2b : b) (2b = b with the
                // exponent + 1: only the high word is selected) and a count of
                // masked products (R = acc - count * t afterwards)
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        const bool m = la[r] > lth[c];
                        const double s = __hiloint2double(static_cast<int>(m ? hi(lx1[c]) : hi(lx0[c])),
                                                          static_cast<int>(lo(lx0[c])));
                        acc[r][c] = __fma_rn(la[r], s, acc[r][c]);
                        cnt[r][c] += m ? 1 : 0;
                    }
                return;
            }
            if constexpr (FORM == 39) {
                // boost as shipped (|u| form): acc0 += a b, u = a b - t, acc1 += |u|
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r) {
                        acc[r][c] = __fma_rn(la[r], lx0[c], acc[r][c]);
                        const double u = __fma_rn(la[r], lx0[c], -lth[c]);
                        acc2[r][c] = __dadd_rn(acc2[r][c], fabs(u));
                    }
                return;
            }
            if constexpr (FORM == 12) {
#pragma unroll
                for (int c = 0; c < TN; ++c)
#pragma unroll
                    for (int r = 0; r < TM; ++r)
                        acc[r][c] = __fma_rn(la[r], la[r] > lth[c] ? lx1[c] : lx0[c], acc[r][c]);
                return;
            }
#pragma unroll
            for (int r = 0; r < TM; ++r)
#pragma unroll
                for (int c = 0; c < TN; ++c)
                    acc[r][c] = __fma_rn(la[r], la[r] > lth[c] ? lx1[c] : lx0[c], acc[r][c]);
        };
        if constexpr (FORM == 9) {
            load(0, na, nth, nx0, nx1);
            for (int it = 0; it < ITERS; it += 2) {
                load((it + 1) & 7, a, th, x0, x1);
                compute(na, nth, nx0, nx1);
                load((it + 2) & 7, na, nth, nx0, nx1);
                compute(a, th, x0, x1);
            }
        } else {
#pragma unroll 2
            for (int it = 0; it < ITERS; ++it) {
                load(it & 7, a, th, x0, x1);
                compute(a, th, x0, x1);
            }
        }
    } else
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int r = 0; r < TM; ++r) asm volatile("" : "+d"(a[r]));
#pragma unroll
        for (int c = 0; c < TN; ++c) asm volatile("" : "+d"(th[c]), "+d"(x0[c]), "+d"(x1[c]));
        if constexpr (FORM == 0) {  // C: row-inner, as the tile kernel writes it (column outer)
#pragma unroll
            for (int c = 0; c < TN; ++c)
#pragma unroll
                for (int r = 0; r < TM; ++r) acc[r][c] = __fma_rn(a[r], a[r] > th[c] ? x1[c] : x0[c], acc[r][c]);
        } else if constexpr (FORM == 1) {  // C: column-inner
#pragma unroll
            for (int r = 0; r < TM; ++r)
#pragma unroll
                for (int c = 0; c < TN; ++c) acc[r][c] = __fma_rn(a[r], a[r] > th[c] ? x1[c] : x0[c], acc[r][c]);
        } else if constexpr (FORM == 2) {  // PTX grouped per column: setp x8, selp lo x8, selp hi x8, fma x8
#pragma unroll
            for (int c = 0; c < TN; ++c) {
                asm volatile(
                    "{\n .reg .pred p<8>; .reg .b32 l<8>, h<8>; .reg .f64 x<8>;\n"
                    " .reg .b32 x0l, x0h, x1l, x1h;\n"
                    " mov.b64 {x0l, x0h}, %9; mov.b64 {x1l, x1h}, %10;\n"
                    " setp.gt.f64 p0, %11, %8; setp.gt.f64 p1, %12, %8; setp.gt.f64 p2, %13, %8; setp.gt.f64 p3, %14, %8;\n"
                    " setp.gt.f64 p4, %15, %8; setp.gt.f64 p5, %16, %8; setp.gt.f64 p6, %17, %8; setp.gt.f64 p7, %18, %8;\n"
                    " selp.b32 l0, x1l, x0l, p0; selp.b32 l1, x1l, x0l, p1; selp.b32 l2, x1l, x0l, p2; selp.b32 l3, x1l, x0l, p3;\n"
                    " selp.b32 l4, x1l, x0l, p4; selp.b32 l5, x1l, x0l, p5; selp.b32 l6, x1l, x0l, p6; selp.b32 l7, x1l, x0l, p7;\n"
                    " selp.b32 h0, x1h, x0h, p0; selp.b32 h1, x1h, x0h, p1; selp.b32 h2, x1h, x0h, p2; selp.b32 h3, x1h, x0h, p3;\n"
                    " selp.b32 h4, x1h, x0h, p4; selp.b32 h5, x1h, x0h, p5; selp.b32 h6, x1h, x0h, p6; selp.b32 h7, x1h, x0h, p7;\n"
                    " mov.b64 x0, {l0, h0}; mov.b64 x1, {l1, h1}; mov.b64 x2, {l2, h2}; mov.b64 x3, {l3, h3};\n"
                    " mov.b64 x4, {l4, h4}; mov.b64 x5, {l5, h5}; mov.b64 x6, {l6, h6}; mov.b64 x7, {l7, h7};\n"
                    " fma.rn.f64 %0, %11, x0, %0; fma.rn.f64 %1, %12, x1, %1; fma.rn.f64 %2, %13, x2, %2; fma.rn.f64 %3, %14, x3, %3;\n"
                    " fma.rn.f64 %4, %15, x4, %4; fma.rn.f64 %5, %16, x5, %5; fma.rn.f64 %6, %17, x6, %6; fma.rn.f64 %7, %18, x7, %7;\n"
                    "}\n"
                    : "+d"(acc[0][c]), "+d"(acc[1][c]), "+d"(acc[2][c]), "+d"(acc[3][c]), "+d"(acc[4][c]),
                      "+d"(acc[5][c]), "+d"(acc[6][c]), "+d"(acc[7][c])
                    : "d"(th[c]), "d"(x0[c]), "d"(x1[c]), "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]),
                      "d"(a[5]), "d"(a[6]), "d"(a[7]));
            }
        } else if constexpr (FORM == 3 || FORM == 4) {
            // compare on the high words only (valid when every a >= 0 has a zero low word):
            // 3: as f32 (FSETP), 4: as s32 (ISETP)
#pragma unroll
            for (int r = 0; r < TM; ++r) ahf[r] = __uint_as_float(hi(a[r]));
#pragma unroll
            for (int c = 0; c < TN; ++c) thf[c] = __uint_as_float(hi(th[c]));
#pragma unroll
            for (int c = 0; c < TN; ++c)
#pragma unroll
                for (int r = 0; r < TM; ++r) {
                    bool m;
                    if constexpr (FORM == 3)
                        m = ahf[r] > thf[c];
                    else
                        m = static_cast<int>(hi(a[r])) > static_cast<int>(hi(th[c]));
                    acc[r][c] = __fma_rn(a[r], m ? x1[c] : x0[c], acc[r][c]);
                }
        } else if constexpr (FORM == 5) {  // DFMA only, a shared per row (the pipe's own rate)
#pragma unroll
            for (int c = 0; c < TN; ++c)
#pragma unroll
                for (int r = 0; r < TM; ++r) acc[r][c] = __fma_rn(a[r], x0[c], acc[r][c]);
        } else if constexpr (FORM == 6) {  // DSETP + 2 FSEL only (no DFMA): select into acc
#pragma unroll
            for (int c = 0; c < TN; ++c)
#pragma unroll
                for (int r = 0; r < TM; ++r) acc[r][c] = a[r] > th[c] ? x1[c] : acc[r][c];
        } else if constexpr (FORM == 7) {  // 2 DFMA per product (the 3-op ordinary discount's pipe load minus the select)
#pragma unroll
            for (int c = 0; c < TN; ++c)
#pragma unroll
                for (int r = 0; r < TM; ++r) acc[r][c] = __fma_rn(a[r], x0[c], __fma_rn(a[r], x1[c], acc[r][c]));
        }
    }
    const long long c1 = clock64();
    double s = 0;
#pragma unroll
    for (int r = 0; r < TM; ++r)
#pragma unroll
        for (int c = 0; c < TN; ++c) s += acc[r][c] + acc2[r][c] + cnt[r][c];
    if (s == 1234.5) out[t] = s;
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
}

template <int FORM>
void run(int sms, int blk, const char* name, double* out, const double* in, long long* cyc) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    kern<FORM><<<sms * blk, 384>>>(out, in, cyc);
    cudaEventRecord(e0);
    kern<FORM><<<sms * blk, 384>>>(out, in, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    // 12 warps per SM = 3 per SMSP, each ITERS * TM * TN warp-products
    printf("%-58s %8.3f ms  %.2f cycles/warp-product/SMSP (clock64, block 0)\n", name, ms,
           double(h[0]) / (double(ITERS) * TM * TN * 3));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out, *in;
    long long* cyc;
    cudaMalloc(&out, 4096 * 8);
    cudaMalloc(&in, 256 * 8);
    cudaMalloc(&cyc, 4096 * 8);
    double h[256];
    for (int i = 0; i < 64; ++i) h[i] = double(i % 10);                 // a: integers 0..9
    for (int i = 0; i < 64; ++i) h[64 + i] = 0.5 + (i * 37 % 64) * 0.13;  // theta
    for (int i = 0; i < 64; ++i) h[128 + i] = 1.0 + i * 1.37;             // x0
    for (int i = 0; i < 64; ++i) h[192 + i] = 0.8 * (1.0 + i * 1.37);     // x1
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    {
        const int blk = 1;
        run<12>(sms, blk, "12 smem-fed, column outer (as the tile kernel)", out, in, cyc);
        run<15>(sms, blk, "15 smem-fed, DFMA only", out, in, cyc);
        run<25>(sms, blk, "25 theta form, PTX block per column", out, in, cyc);
        run<26>(sms, blk, "26 theta form, PTX block per row", out, in, cyc);
        run<27>(sms, blk, "27 int64 compare (ALU) for every product", out, in, cyc);
        run<28>(sms, blk, "28 int64 compare for 1 column of 4", out, in, cyc);
        run<29>(sms, blk, "29 int64 compare for 2 columns of 4", out, in, cyc);
        run<30>(sms, blk, "30 int64 compare for 2 rows of 8", out, in, cyc);
        run<31>(sms, blk, "31 col 3 Y (IMAD compare + IMAD select)", out, in, cyc);
        run<32>(sms, blk, "32 col 2 X (ISETP), col 3 Y", out, in, cyc);
        run<33>(sms, blk, "33 all Y", out, in, cyc);
        run<34>(sms, blk, "34 all I (DADD sign + IMAD select)", out, in, cyc);
        run<35>(sms, blk, "35 col 3 I", out, in, cyc);
        run<36>(sms, blk, "36 cols 2-3 I", out, in, cyc);
        run<37>(sms, blk, "37 col 1 I, col 3 Y", out, in, cyc);
        run<38>(sms, blk, "38 boost theta form (DSETP, FSEL hi, DFMA, count)", out, in, cyc);
        run<39>(sms, blk, "39 boost |u| form as shipped (2 DFMA + DADD)", out, in, cyc);
        if (getenv("ALLFORMS")) {
        run<18>(sms, blk, "18 P3: ISETP hi + DFMA x0 + @P DFMA d", out, in, cyc);
        run<19>(sms, blk, "19 P3 grouped per column (PTX)", out, in, cyc);
        run<20>(sms, blk, "20 P3 with DSETP", out, in, cyc);
        run<21>(sms, blk, "21 2 DFMA per product", out, in, cyc);
        run<22>(sms, blk, "22 HSETP2 (2 masks/instr) + 2 FSEL + DFMA", out, in, cyc);
        run<23>(sms, blk, "23 HSETP2 + FSEL only", out, in, cyc);
        run<24>(sms, blk, "24 ISETP + SEL hi(a) + 2 DFMA", out, in, cyc);
        }
        if (getenv("ALLFORMS")) {
        run<8>(sms, blk, "8 smem-fed, row outer", out, in, cyc);
        run<9>(sms, blk, "9 smem-fed, next k loaded before this k's compute", out, in, cyc);
        run<10>(sms, blk, "10 B from smem, a in registers", out, in, cyc);
        run<11>(sms, blk, "11 a from smem, B in registers", out, in, cyc);
        run<12>(sms, blk, "12 smem-fed, column outer (as the tile kernel)", out, in, cyc);
        run<13>(sms, blk, "13 smem-fed, high-word compare as f32 (FSETP)", out, in, cyc);
        run<14>(sms, blk, "14 smem-fed, high-word compare as s32 (ISETP)", out, in, cyc);
        run<15>(sms, blk, "15 smem-fed, DFMA only", out, in, cyc);
        run<16>(sms, blk, "16 smem-fed, DSETP + 2 FSEL only", out, in, cyc);
        run<17>(sms, blk, "17 smem-fed, FSETP + 2 FSEL only", out, in, cyc);
        }
    }
    return 0;
}
