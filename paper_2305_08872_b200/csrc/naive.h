// naive.h — the per-element device executor (naive.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/amlt_gpu.h"

namespace amltk {

// Statement-level addressing: element (i, k) of A is A[i*sai + k*sak], and
// likewise for B (k, j), R (i, j), thres (i, j) and dis (j). Offsets are
// already applied for the bounds' origin; i, j, k run from 0.
struct NaiveParams {
    const void* A;
    const void* B;
    void* R;
    const void* thres;  // null: tconst
    const void* dis;
    int64_t sai, sak, sbk, sbj, sri, srj, t_si, t_sj, d_sj;
    int64_t M, N, K;
    double tconst;
    int accumulate;
};

cudaError_t launch_naive(const NaiveParams& p, int body, int dtype, int num_sms, cudaStream_t s);

}  // namespace amltk
