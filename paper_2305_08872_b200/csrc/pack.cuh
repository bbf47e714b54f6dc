// pack.cuh — operand packing for the layouts the tiled kernels do not stage
// directly.
//
// The kernels read A along k and B / R along j (row-major A[i][k], B[k][j],
// R[i][j]). Every other layout the reference accepts — the transposed
// statements A[k][i] / B[j][k] (presets -atb/-abt/-atbt) and col-major
// storage (matrix.hpp:10) — is first packed into a dense row-major workspace,
// exactly as the reference's packing absorbs orientation and storage order
// (packing.hpp:11-18,44-46, src/packing.cpp:5-45). R in a layout other than
// j-contiguous is packed, updated, and unpacked back. Packing is an
// HBM-bound transpose through shared memory, coalesced on both sides; it is
// a small fraction of a compute-bound subtask (O(MK + KN) bytes vs O(MNK)
// work).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace amltk {

struct PackParams {
    const void* src;
    void* dst;
    int64_t rows, cols;  // logical (statement) extents
    int64_t s0, s1;      // element strides of the strided side along rows / cols
    int64_t ld;          // leading dimension of the dense row-major side
    int32_t unpack;      // 0: strided -> dense, 1: dense -> strided
};

// 32 x 32 tiles staged through shared memory; each side is read / written in
// its own contiguous direction (whichever of s0 / s1 is 1, else rows).
template <typename T>
__global__ void __launch_bounds__(256) mmlt_pack_kernel(const PackParams p) {
    __shared__ T tile[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32;
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    const bool strided_rows_fast = p.s0 == 1 && p.s1 != 1;  // strided side contiguous along rows
    const T* src = static_cast<const T*>(p.src);
    T* dst = static_cast<T*>(p.dst);
    // load
    for (int y = ty; y < 32; y += 8) {
        int64_t r, c;
        if (!p.unpack && strided_rows_fast) {
            r = r0 + tx;
            c = c0 + y;
        } else {
            r = r0 + y;
            c = c0 + tx;
        }
        if (r < p.rows && c < p.cols) {
            const T v = p.unpack ? src[r * p.ld + c] : src[r * p.s0 + c * p.s1];
            tile[r - r0][c - c0] = v;
        }
    }
    __syncthreads();
    // store
    for (int y = ty; y < 32; y += 8) {
        int64_t r, c;
        if (p.unpack && strided_rows_fast) {
            r = r0 + tx;
            c = c0 + y;
        } else {
            r = r0 + y;
            c = c0 + tx;
        }
        if (r < p.rows && c < p.cols) {
            const T v = tile[r - r0][c - c0];
            if (p.unpack)
                dst[r * p.s0 + c * p.s1] = v;
            else
                dst[r * p.ld + c] = v;
        }
    }
}

template <typename T>
cudaError_t launch_pack(const PackParams& p, cudaStream_t s) {
    if (p.rows <= 0 || p.cols <= 0) return cudaSuccess;
    dim3 grid(static_cast<unsigned>((p.cols + 31) / 32), static_cast<unsigned>((p.rows + 31) / 32));
    if (grid.y > 65535) return cudaErrorInvalidValue;
    mmlt_pack_kernel<T><<<grid, dim3(32, 8), 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace amltk
