// matrix_file.cpp — the reference's AMLT binary matrix format, read straight
// into host or device buffers of the kernel dtype.
//
// Format (README.md:146-157, src/matrix.cpp:64-114): 24-byte header — magic
// "AMLT", u32 rows, u32 cols (little endian), u8 storage order (0 row-major,
// 1 col-major), 11 zero bytes — then rows*cols little-endian f64 values in
// storage order. Files are the input side of the hot path (the reference
// CLI's --a-file / --b-file); reading converts to f32 / i32 when the plan
// computes in those types and uploads in chunks through a pinned buffer.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/amlt_gpu.h"

namespace {

thread_local std::string g_err;

constexpr char kMagic[4] = {'A', 'M', 'L', 'T'};
constexpr size_t kHeader = 24;

uint32_t get_u32(const unsigned char* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}
void put_u32(unsigned char* p, uint32_t v) {
    for (int i = 0; i < 4; ++i) p[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
}

amlt_status fail(amlt_status st, const std::string& m) {
    g_err = m;
    return st;
}

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

amlt_status read_header(FILE* f, const char* path, int64_t* rows, int64_t* cols, int* order) {
    unsigned char h[kHeader];
    if (std::fread(h, 1, kHeader, f) != kHeader || std::memcmp(h, kMagic, 4) != 0)
        return fail(AMLT_ERR_ENGINE, std::string("'") + path + "' is not a matrix file (bad magic)");
    if (h[12] > 1) return fail(AMLT_ERR_ENGINE, std::string("'") + path + "' has an unknown storage order");
    *rows = get_u32(h + 4);
    *cols = get_u32(h + 8);
    *order = h[12];
    return AMLT_OK;
}

int esize(int dt) { return dt == AMLT_F64 ? 8 : 4; }

void convert(const double* src, void* dst, size_t n, int dt) {
    if (dt == AMLT_F64) {
        std::memcpy(dst, src, n * 8);
    } else if (dt == AMLT_F32) {
        float* d = static_cast<float*>(dst);
        for (size_t i = 0; i < n; ++i) d[i] = static_cast<float>(src[i]);
    } else {
        int32_t* d = static_cast<int32_t*>(dst);
        for (size_t i = 0; i < n; ++i) d[i] = static_cast<int32_t>(src[i]);
    }
}

}  // namespace

extern "C" {

const char* amlt_matrix_file_last_error(void) { return g_err.c_str(); }

amlt_status amlt_matrix_file_info(const char* path, int64_t* rows, int64_t* cols, int* order) {
    if (!path || !rows || !cols || !order) return AMLT_ERR_INVALID_ARGUMENT;
    File fl;
    fl.f = std::fopen(path, "rb");
    if (!fl.f) return fail(AMLT_ERR_ENGINE, std::string("cannot open '") + path + "'");
    return read_header(fl.f, path, rows, cols, order);
}

amlt_status amlt_matrix_file_read(const char* path, void* dst, int dtype, int dst_on_device) {
    if (!path || !dst || dtype < AMLT_F64 || dtype > AMLT_I32) return AMLT_ERR_INVALID_ARGUMENT;
    File fl;
    fl.f = std::fopen(path, "rb");
    if (!fl.f) return fail(AMLT_ERR_ENGINE, std::string("cannot open '") + path + "'");
    int64_t rows, cols;
    int order;
    amlt_status st = read_header(fl.f, path, &rows, &cols, &order);
    if (st != AMLT_OK) return st;
    const size_t n = size_t(rows) * size_t(cols);
    const size_t chunk = size_t(1) << 22;  // 4 Mi values per pass
    std::vector<double> buf(std::min(n, chunk));
    void* pinned = nullptr;
    const int es = esize(dtype);
    if (dst_on_device && cudaMallocHost(&pinned, std::min(n, chunk) * es + 16) != cudaSuccess)
        return fail(AMLT_ERR_CUDA, "cudaMallocHost failed");
    amlt_status out = AMLT_OK;
    for (size_t off = 0; off < n; off += chunk) {
        const size_t m = std::min(chunk, n - off);
        if (std::fread(buf.data(), 8, m, fl.f) != m) {
            out = fail(AMLT_ERR_ENGINE, std::string("'") + path + "' is truncated");
            break;
        }
        if (dst_on_device) {
            convert(buf.data(), pinned, m, dtype);
            if (cudaMemcpy(static_cast<char*>(dst) + off * es, pinned, m * es,
                           cudaMemcpyHostToDevice) != cudaSuccess) {
                out = fail(AMLT_ERR_CUDA, "cudaMemcpy to device failed");
                break;
            }
        } else {
            convert(buf.data(), static_cast<char*>(dst) + off * es, m, dtype);
        }
    }
    if (pinned) cudaFreeHost(pinned);
    return out;
}

amlt_status amlt_matrix_file_write(const char* path, const void* src, int64_t rows, int64_t cols,
                                   int order, int dtype, int src_on_device) {
    if (!path || (!src && rows * cols > 0) || rows < 0 || cols < 0 || order < 0 || order > 1 ||
        rows > 0xffffffffLL || cols > 0xffffffffLL || dtype < AMLT_F64 || dtype > AMLT_I32)
        return AMLT_ERR_INVALID_ARGUMENT;
    const size_t n = size_t(rows) * size_t(cols);
    const int es = esize(dtype);
    std::vector<unsigned char> host;
    const unsigned char* p = static_cast<const unsigned char*>(src);
    if (src_on_device && n) {
        host.resize(n * es);
        if (cudaMemcpy(host.data(), src, n * es, cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(AMLT_ERR_CUDA, "cudaMemcpy from device failed");
        p = host.data();
    }
    File fl;
    fl.f = std::fopen(path, "wb");
    if (!fl.f) return fail(AMLT_ERR_ENGINE, std::string("cannot open '") + path + "' for writing");
    unsigned char h[kHeader] = {0};
    std::memcpy(h, kMagic, 4);
    put_u32(h + 4, static_cast<uint32_t>(rows));
    put_u32(h + 8, static_cast<uint32_t>(cols));
    h[12] = static_cast<unsigned char>(order);
    if (std::fwrite(h, 1, kHeader, fl.f) != kHeader) return fail(AMLT_ERR_ENGINE, "write failed");
    std::vector<double> d(std::min<size_t>(n, size_t(1) << 20));
    for (size_t off = 0; off < n; off += d.size()) {
        const size_t m = std::min(d.size(), n - off);
        for (size_t i = 0; i < m; ++i) {
            const unsigned char* e = p + (off + i) * es;
            if (dtype == AMLT_F64) std::memcpy(&d[i], e, 8);
            else if (dtype == AMLT_F32) {
                float v;
                std::memcpy(&v, e, 4);
                d[i] = v;
            } else {
                int32_t v;
                std::memcpy(&v, e, 4);
                d[i] = v;
            }
        }
        if (std::fwrite(d.data(), 8, m, fl.f) != m) return fail(AMLT_ERR_ENGINE, "write failed");
    }
    return AMLT_OK;
}

uint64_t amlt_operand_seed(uint64_t seed, const char* name) {
    // seed ^ fnv1a(name): the per-array seed of make_task_data
    // (reference src/engine.cpp:17-24,147).
    uint64_t h = 1469598103934665603ull;
    for (const unsigned char* c = reinterpret_cast<const unsigned char*>(name ? name : ""); *c; ++c) {
        h ^= *c;
        h *= 1099511628211ull;
    }
    return seed ^ h;
}

amlt_status amlt_gen_matrix(uint64_t seed, int64_t rows, int64_t cols, int order, int mode,
                            void* dst, int dtype, int dst_on_device) {
    // The reference's deterministic inputs (src/matrix.cpp:20-37): mt19937_64
    // over seed_seq{seed, rows, cols, order, mode}; IntValued (mode 0) draws
    // uniform ints in [-8, 8], Real (mode 1) uniform doubles in [0, 1). The
    // same standard-library engine and distributions are used, so the buffers
    // match the reference's bit for bit under the same C++ runtime.
    if (!dst || rows < 0 || cols < 0 || order < 0 || order > 1 || mode < 0 || mode > 1 ||
        dtype < AMLT_F64 || dtype > AMLT_I32)
        return AMLT_ERR_INVALID_ARGUMENT;
    std::seed_seq seq{seed, static_cast<uint64_t>(rows), static_cast<uint64_t>(cols),
                      static_cast<uint64_t>(order), static_cast<uint64_t>(mode)};
    std::mt19937_64 rng(seq);
    const size_t n = size_t(rows) * size_t(cols);
    const size_t chunk = size_t(1) << 22;
    const int es = esize(dtype);
    std::vector<double> buf(std::min(n, chunk));
    std::vector<unsigned char> conv(dst_on_device ? buf.size() * es : 0);
    std::uniform_int_distribution<int> idist(-8, 8);
    std::uniform_real_distribution<double> rdist(0.0, 1.0);
    for (size_t off = 0; off < n; off += chunk) {
        const size_t m = std::min(chunk, n - off);
        if (mode == 0)
            for (size_t i = 0; i < m; ++i) buf[i] = static_cast<double>(idist(rng));
        else
            for (size_t i = 0; i < m; ++i) buf[i] = rdist(rng);
        if (dst_on_device) {
            convert(buf.data(), conv.data(), m, dtype);
            if (cudaMemcpy(static_cast<char*>(dst) + off * es, conv.data(), m * es,
                           cudaMemcpyHostToDevice) != cudaSuccess)
                return fail(AMLT_ERR_CUDA, "cudaMemcpy to device failed");
        } else {
            convert(buf.data(), static_cast<char*>(dst) + off * es, m, dtype);
        }
    }
    return AMLT_OK;
}

}  // extern "C"
