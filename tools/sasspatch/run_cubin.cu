// Scratch harness (not product code): runs one thetabench kernel from a
// (possibly patched) cubin through the driver API, 1 CTA of 384 threads per
// SM as tools/thetabench.cu does, and prints cycles per warp-product.
//   nvcc -o run_cubin tools/sasspatch/run_cubin.cu -lcuda
//   ./run_cubin tb.cubin _Z4kernILi12EEvPdPKdPx
#include <cuda.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
    std::fprintf(stderr, "%s: %s\n", #x, s); return 1; } } while (0)

int main(int argc, char** argv) {
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    CUcontext ctx;
    CK(cuDevicePrimaryCtxRetain(&ctx, dev));
    CK(cuCtxSetCurrent(ctx));
    CUmodule mod;
    CK(cuModuleLoad(&mod, argv[1]));
    CUfunction f;
    CK(cuModuleGetFunction(&f, mod, argv[2]));
    int sms;
    CK(cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev));
    CUdeviceptr out, in, cyc;
    CK(cuMemAlloc(&out, 4096 * 8));
    CK(cuMemAlloc(&in, 256 * 8));
    CK(cuMemAlloc(&cyc, 4096 * 8));
    std::vector<double> h(256);
    for (int i = 0; i < 64; ++i) h[i] = double(i % 10);
    for (int i = 0; i < 64; ++i) h[64 + i] = 0.5 + (i * 37 % 64) * 0.13;
    for (int i = 0; i < 64; ++i) h[128 + i] = 1.0 + i * 1.37;
    for (int i = 0; i < 64; ++i) h[192 + i] = 0.8 * (1.0 + i * 1.37);
    CK(cuMemcpyHtoD(in, h.data(), 256 * 8));
    void* args[] = {&out, &in, &cyc};
    CUevent e0, e1;
    CK(cuEventCreate(&e0, 0));
    CK(cuEventCreate(&e1, 0));
    double best = 1e30, best_cyc = 0;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cuEventRecord(e0, 0));
        CK(cuLaunchKernel(f, sms, 1, 1, 384, 1, 1, 0, 0, args, nullptr));
        CK(cuEventRecord(e1, 0));
        CK(cuEventSynchronize(e1));
        float ms;
        CK(cuEventElapsedTime(&ms, e0, e1));
        long long c;
        CK(cuMemcpyDtoH(&c, cyc, sizeof(c)));
        if (ms < best) { best = ms; best_cyc = double(c); }
    }
    std::vector<double> o(4096);
    CK(cuMemcpyDtoH(o.data(), out, 4096 * 8));
    double sum = 0;
    for (double v : o) sum += v;
    // 8 x 4 micro-tile, 4096 iterations, 12 warps per SM = 3 per SMSP
    std::printf("%s %s: %.3f ms, %.2f cycles/warp-product/SMSP, checksum %.17g\n", argv[1], argv[2], best,
                best_cyc / (4096.0 * 32 * 3), sum);
    return 0;
}
