// variants.h — registry of compiled tile variants (host side).
//
// One entry per (body, dtype, tile shape) kernel instantiation. This is the
// GPU counterpart of the reference's kernel planner (choose_kernel_shape /
// register_ledger, src/kernel_plan.cpp:45-104): instead of one register
// footprint picked from a CPU register budget, every feasible CTA/thread tile
// is compiled ahead of time and the runtime tuner measures among them.
#pragma once

#include <cuda_runtime.h>

#include <deque>
#include <mutex>
#include <vector>

#include "mmlt_kernel.cuh"
#include "pack.cuh"

namespace amltk {

using LaunchFn = cudaError_t (*)(const KParams&, dim3 grid, cudaStream_t);
// Tile kernels also take the two TMA descriptors (A box BK x BM, B box
// BN x BK); element-staged variants receive zeroed descriptors.
using TileLaunchFn = cudaError_t (*)(const KParams&, const CUtensorMap& a, const CUtensorMap& b,
                                     dim3 grid, cudaStream_t);

struct VariantDesc {
    int body = 0;
    int dtype = 0;
    int bm = 0, bn = 0, bk = 0, tm = 0, tn = 0;
    int threads = 0, stages = 0, smem = 0, minb = 1;
    bool vec = true;  // TMA staging (needs 16-byte aligned operands and strides)
    bool tc = false;  // tensor-core (DMMA) variant
    bool tout = false;  // per-output threshold state (T indexed by i or (i, j))
    bool emulated = false;  // f64 via int8 tensor cores: tuner candidate only on opt-in
    int64_t max_k = 0;      // largest K range the variant accepts (0: any)
    const char* name = "";
    const void* func = nullptr;
    TileLaunchFn launch = nullptr;
    // Variants with their own staging (tcgen05 3xTF32 GEMM): the whole
    // subtask is run(), with ws_bytes() of context workspace.
    // B's preparation (split / slices) sits at the front of the workspace and
    // is reused across the row bands of one call (b_ready); prep_id names its
    // format, prep_b computes it alone (before a timed trial).
    size_t (*ws_bytes)(const KParams&) = nullptr;
    cudaError_t (*run)(const KParams&, void* ws, bool b_ready, cudaStream_t) = nullptr;
    cudaError_t (*prep_b)(const KParams&, void* ws, cudaStream_t) = nullptr;
    int prep_id = 0;
    // run() variants that accept K segments (KParams splits / kslice / work,
    // partials reduced in segment order afterwards like the tile variants)
    bool splittable = false;
    // the epilogue honours KParams::r_zero and stores R with plain global
    // loads / stores (R may be mapped host memory)
    bool r_overwrite = false;
    // prep_b / run honour KParams::plane_k0 / plane_kdim: B can be prepared
    // K panel by K panel into one whole-K preparation as the panels land
    bool prep_panels = false;
};

// Per (body, dtype) helpers that are not tile variants.
struct BodyAux {
    int body = 0;
    int dtype = 0;
    // Generated bodies: launched through the kernel handles below
    // (assign == nullptr); naive_func is their per-element executor.
    const void* naive_func = nullptr;
    LaunchFn assign = nullptr;  // "=" statements: last k wins
    LaunchFn reduce = nullptr;  // split-K ordered reduction into R
    cudaError_t (*pack)(const PackParams&, cudaStream_t) = nullptr;  // layout packing
    const void* pack_func = nullptr;
    const void* assign_func = nullptr;
    const void* reduce_func = nullptr;
};

// Append-only (run-time compiled bodies add entries): deques keep the
// addresses of existing entries stable.
struct Registry {
    std::deque<VariantDesc> variants;
    std::deque<BodyAux> aux;
};

// The process-wide registry (amlt_gpu.cu); appends take registry_mutex().
Registry& registry_mut();
std::mutex& registry_mutex();

// Launch a tile variant / helper kernel whether it is a compiled-in template
// (launch function) or a run-time compiled kernel handle (func only).
inline cudaError_t launch_tile_any(const VariantDesc& v, const KParams& p, const CUtensorMap& a,
                                   const CUtensorMap& b, dim3 grid, cudaStream_t s) {
    if (v.launch) return v.launch(p, a, b, grid, s);
    if (!v.func) return cudaErrorInvalidDeviceFunction;
    void* args[3] = {const_cast<KParams*>(&p), const_cast<CUtensorMap*>(&a),
                     const_cast<CUtensorMap*>(&b)};
    return cudaLaunchKernel(v.func, grid, dim3(v.threads), args, static_cast<size_t>(v.smem), s);
}
inline cudaError_t launch_helper_any(LaunchFn fn, const void* func, const KParams& p, dim3 grid,
                                     cudaStream_t s) {
    if (fn) return fn(p, grid, s);
    if (!func) return cudaErrorInvalidDeviceFunction;
    void* args[1] = {const_cast<KParams*>(&p)};
    return cudaLaunchKernel(func, grid, dim3(256), args, 0, s);
}

// Defined once per (body, dtype) translation unit (kernels_inst.cu) and by
// the DMMA GEMM unit; collected by registry() in amlt_gpu.cu.
void register_all(Registry& reg);

template <class Cfg, class Body, typename T, int TM, int TN, int WR, int WC, int BK, int STAGES,
          int LOAD, int MINB>
cudaError_t launch_tile(const KParams& p, const CUtensorMap& a, const CUtensorMap& b, dim3 grid,
                        cudaStream_t s) {
    mmlt_tile_kernel<Body, T, TM, TN, WR, WC, BK, STAGES, LOAD, MINB>
        <<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(p, a, b);
    return cudaGetLastError();
}

template <class Body, typename T>
cudaError_t launch_assign(const KParams& p, dim3 grid, cudaStream_t s) {
    mmlt_assign_kernel<Body, T><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_reduce(const KParams& p, dim3 grid, cudaStream_t s) {
    mmlt_splitk_reduce<T><<<grid, 256, 0, s>>>(p);
    return cudaGetLastError();
}

template <class Body, typename T, int TM, int TN, int WR, int WC, int BK, int STAGES, int LOAD,
          int MINB>
void add_variant(Registry& reg, int body, int dtype, const char* name) {
    using Cfg = MmltTile<Body, T, TM, TN, WR, WC, BK, STAGES, LOAD, MINB>;
    // Register budget guard: accumulators (two-level bodies keep a second
    // set) must leave room for operands; larger tiles are not instantiated.
    constexpr int acc_regs =
        TM * TN * Body::NACC * (Body::TWO_LEVEL ? 2 : 1) * (int)(sizeof(typename Body::Acc) / 4);
    if constexpr (acc_regs <= 136) {
        VariantDesc v;
        v.body = body;
        v.dtype = dtype;
        v.bm = Cfg::BM;
        v.bn = Cfg::BN;
        v.bk = BK;
        v.tm = TM;
        v.tn = TN;
        v.threads = Cfg::THREADS;
        v.stages = STAGES;
        v.smem = Cfg::SMEM_BYTES;
        v.minb = MINB;
        v.vec = (LOAD & LOAD_TMA) != 0;
        v.tout = (LOAD & LOAD_TOUT) != 0;
        v.r_overwrite = true;
        v.name = name;
        v.func = reinterpret_cast<const void*>(
            &mmlt_tile_kernel<Body, T, TM, TN, WR, WC, BK, STAGES, LOAD, MINB>);
        v.launch = &launch_tile<Cfg, Body, T, TM, TN, WR, WC, BK, STAGES, LOAD, MINB>;
        reg.variants.push_back(v);
    }
}

}  // namespace amltk
