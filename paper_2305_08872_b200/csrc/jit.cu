// jit.cu — run-time compiled bodies (AMLT_BODY_GENERIC).
//
// The fixed bodies cover the five BASELINE statements and q3; the reference
// recognises many more multiply-accumulate-like statements (its TaskGen
// draws them at random: aux leaves u[i], v[j], W[i][j], scalars, constants,
// + - * / and comparisons; recognize.cpp:84-166, test_support.hpp) and runs
// them through its pseudo-program interpreter (run_instrs,
// kernel_exec.cpp:63-126). Here such a statement becomes a Body struct whose
// step evaluates the statement term node by node — one correctly rounded
// IEEE operation per syntax-tree node, comparisons as 1 / 0, exactly the
// reference's naive evaluation (naive.cpp:85-117) — and is compiled by NVRTC
// for sm_100a into the same tile kernels as the fixed bodies (TMA staging,
// split-K, grouped raster), plus the "=" and per-element kernels. Nothing is
// interpreted on the device.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>
#include <nvrtc.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <type_traits>
#include <vector>

#include "jit.h"

namespace amltk {

namespace {

const char kKernelHeader[] =
#include "mmlt_kernel_src.inc"
    ;

// NVRTC through dlopen: the library is only needed when a generated body is
// planned.
struct Nvrtc {
    decltype(&nvrtcCreateProgram) create = nullptr;
    decltype(&nvrtcDestroyProgram) destroy = nullptr;
    decltype(&nvrtcCompileProgram) compile = nullptr;
    decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
    decltype(&nvrtcGetCUBIN) cubin = nullptr;
    decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
    decltype(&nvrtcGetProgramLog) log = nullptr;
    decltype(&nvrtcAddNameExpression) add_name = nullptr;
    decltype(&nvrtcGetLoweredName) lowered = nullptr;
    decltype(&nvrtcGetErrorString) error = nullptr;
    std::string why;
};

const Nvrtc& nvrtc() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                                 "/usr/local/cuda/lib64/libnvrtc.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
            if (h) break;
        }
        if (!h) {
            n.why = "libnvrtc.so.12 not found (needed to compile generated bodies)";
            return;
        }
        auto sym = [&](auto& fn, const char* s) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, s));
            if (!fn && n.why.empty()) n.why = std::string("libnvrtc lacks ") + s;
        };
        sym(n.create, "nvrtcCreateProgram");
        sym(n.destroy, "nvrtcDestroyProgram");
        sym(n.compile, "nvrtcCompileProgram");
        sym(n.cubin_size, "nvrtcGetCUBINSize");
        sym(n.cubin, "nvrtcGetCUBIN");
        sym(n.log_size, "nvrtcGetProgramLogSize");
        sym(n.log, "nvrtcGetProgramLog");
        sym(n.add_name, "nvrtcAddNameExpression");
        sym(n.lowered, "nvrtcGetLoweredName");
        sym(n.error, "nvrtcGetErrorString");
    });
    if (!n.why.empty()) throw TaskError(AMLT_ERR_ENGINE, n.why);
    return n;
}

// Tile shapes compiled for a generated body (a subset of the fixed bodies'
// set: the tuner still measures among them).
struct Shape {
    int tm, tn, wr, wc, bk, stages, load, minb;
    const char* name;
};
constexpr int kTma = 1, kElem = 0, kTout = 2;
const Shape kShapesF64[] = {
    {4, 4, 8, 1, 16, 3, kTma, 2, "t4x4_w8x1"},
    {4, 4, 4, 1, 16, 4, kTma, 3, "t4x4_w4x1"},
    {4, 2, 4, 1, 16, 4, kTma, 4, "t4x2_w4x1"},
    {4, 4, 8, 1, 16, 3, kElem, 2, "t4x4_w8x1_u"},
};
const Shape kShapesF32[] = {
    {8, 4, 8, 1, 32, 3, kTma, 1, "t8x4_w8x1"},
    {4, 4, 8, 1, 32, 3, kTma, 2, "t4x4_w8x1"},
    {4, 4, 4, 1, 32, 4, kTma, 3, "t4x4_w4x1"},
    {4, 4, 8, 1, 32, 3, kElem, 2, "t4x4_w8x1_u"},
};
constexpr int kNumShapes = 4;

const char* ctype(int dtype) { return dtype == AMLT_F64 ? "double" : "float"; }

std::string key_of(const RecognizedTask& rt, int dtype) {
    std::string k = std::to_string(dtype) + "|" + rt.expr + "|";
    for (int c : rt.aux_class) k += std::to_string(c) + ",";
    return k;
}

bool has_at(const RecognizedTask& rt) {
    for (int c : rt.aux_class)
        if (c == AMLT_LEAF_VEC_I || c == AMLT_LEAF_MAT_IJ) return true;
    return false;
}

// Per-output aux state (leaves indexed by i or (i, j)) needs registers: the
// 256-thread tiles then drop their two-CTAs-per-SM bound instead of spilling.
int minb_of(const Shape& sh, bool tout) { return tout && sh.wr * sh.wc * 32 >= 256 ? 1 : sh.minb; }

std::string tile_name_expr(const Shape& sh, int dtype, bool tout) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "amltk::mmlt_tile_kernel<amltk::BodyGen, %s, %d, %d, %d, %d, %d, %d, %d, %d>",
                  ctype(dtype), sh.tm, sh.tn, sh.wr, sh.wc, sh.bk, sh.stages,
                  sh.load | (tout ? kTout : 0), minb_of(sh, tout));
    return buf;
}

// On-disk cubin cache, so a generated body compiles once per machine rather
// than once per process: $AMLT_GPU_JIT_CACHE (a directory; "0" disables),
// else $XDG_CACHE_HOME/amlt_gpu or ~/.cache/amlt_gpu. Entries are keyed by a
// 64-bit FNV-1a hash of the full source (header included) and verified
// against the stored source text before use.
uint64_t fnv1a64(const std::string& s) {
    uint64_t h = 1469598103934665603ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 1099511628211ull;
    }
    return h;
}

std::string disk_cache_path(const std::string& src) {
    const char* env = std::getenv("AMLT_GPU_JIT_CACHE");
    std::string dir;
    if (env && *env) {
        if (std::string(env) == "0") return "";
        dir = env;
    } else if (const char* x = std::getenv("XDG_CACHE_HOME"); x && *x) {
        dir = std::string(x) + "/amlt_gpu";
    } else if (const char* h = std::getenv("HOME"); h && *h) {
        dir = std::string(h) + "/.cache/amlt_gpu";
    } else {
        return "";
    }
    std::string cur;
    for (size_t i = 0; i <= dir.size(); ++i)  // mkdir -p
        if (i == dir.size() || (dir[i] == '/' && i > 0)) {
            cur = dir.substr(0, i);
            mkdir(cur.c_str(), 0755);
        }
    char name[64];
    std::snprintf(name, sizeof(name), "/jit-%016llx.bin", static_cast<unsigned long long>(fnv1a64(src)));
    return dir + name + "|" + src;  // the source rides along for verification
}

// File layout: u64 source length, source, u64 name count, (u64 len, name)*,
// u64 cubin length, cubin.
bool disk_cache_read(const std::string& key, size_t n_names, std::vector<char>* cubin,
                     std::vector<std::string>* lowered) {
    const size_t bar = key.find('|');
    const std::string path = key.substr(0, bar), src = key.substr(bar + 1);
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) return false;
    auto rd_u64 = [&](uint64_t* v) { return std::fread(v, 8, 1, f) == 1; };
    auto rd_str = [&](std::string* out) {
        uint64_t n = 0;
        if (!rd_u64(&n) || n > (1ull << 28)) return false;
        out->resize(n);
        return n == 0 || std::fread(&(*out)[0], 1, n, f) == n;
    };
    bool ok = false;
    std::string stored;
    uint64_t names = 0, nc = 0;
    if (rd_str(&stored) && stored == src && rd_u64(&names) && names == n_names) {
        lowered->assign(names, "");
        ok = true;
        for (auto& l : *lowered) ok = ok && rd_str(&l);
        if (ok && rd_u64(&nc) && nc > 0 && nc < (1ull << 30)) {
            cubin->resize(nc);
            ok = std::fread(cubin->data(), 1, nc, f) == nc;
        } else {
            ok = false;
        }
    }
    std::fclose(f);
    return ok;
}

void disk_cache_write(const std::string& key, const std::vector<char>& cubin,
                      const std::vector<std::string>& lowered) {
    const size_t bar = key.find('|');
    const std::string path = key.substr(0, bar), src = key.substr(bar + 1);
    const std::string tmp = path + ".tmp" + std::to_string(static_cast<long long>(getpid()));
    FILE* f = std::fopen(tmp.c_str(), "wb");
    if (!f) return;
    auto wr_u64 = [&](uint64_t v) { std::fwrite(&v, 8, 1, f); };
    auto wr_str = [&](const std::string& s) {
        wr_u64(s.size());
        std::fwrite(s.data(), 1, s.size(), f);
    };
    wr_str(src);
    wr_u64(lowered.size());
    for (const auto& l : lowered) wr_str(l);
    wr_u64(cubin.size());
    std::fwrite(cubin.data(), 1, cubin.size(), f);
    const bool ok = std::fflush(f) == 0;
    std::fclose(f);
    if (ok) std::rename(tmp.c_str(), path.c_str());  // atomic publish
    else std::remove(tmp.c_str());
}

struct Cache {
    std::mutex m;
    std::map<std::string, JitBody> bodies;
    std::deque<std::string> names;  // stable storage for VariantDesc::name
};
Cache& cache() {
    static Cache c;
    return c;
}

}  // namespace

std::string jit_source(const RecognizedTask& rt, int dtype) {
    if (dtype != AMLT_F64 && dtype != AMLT_F32)
        throw TaskError(AMLT_ERR_UNSUPPORTED, "generated bodies compute in f64 or f32");
    const size_t nv = rt.aux_names.size();
    std::string s;
    s += "// generated body for: R (+)= " + rt.expr + "\n";
    s += kKernelHeader;
    s += "\nnamespace amltk {\nstruct BodyGen {\n";
    s += std::string("    using T = ") + ctype(dtype) + ";\n";
    s += "    using Acc = T;\n    static constexpr int NACC = 1;\n    static constexpr bool TWO_LEVEL = false;\n";
    s += std::string("    static constexpr bool HAS_AT = ") + (has_at(rt) ? "true" : "false") + ";\n";
    s += "    struct Col {\n        T v[" + std::to_string(nv ? nv : 1) + "];\n    };\n";
    s += "    __device__ static __forceinline__ Col col(const KParams& p, int64_t j) {\n        Col c;\n";
    for (size_t q = 0; q < nv; ++q) {
        const std::string Q = std::to_string(q);
        if (rt.aux_class[q] == AMLT_LEAF_CONSTANT || rt.aux_class[q] == AMLT_LEAF_VEC_J)
            s += "        c.v[" + Q + "] = ldg_elem<T>(p.gaux[" + Q + "], j * p.gaux_sj[" + Q + "]);\n";
        else
            s += "        c.v[" + Q + "] = T(0);\n";
    }
    if (!nv) s += "        c.v[0] = T(0);\n";
    s += "        return c;\n    }\n";
    s += "    __device__ static __forceinline__ Col at(Col c, const KParams& p, int64_t i, int64_t j) {\n";
    for (size_t q = 0; q < nv; ++q) {
        const std::string Q = std::to_string(q);
        if (rt.aux_class[q] == AMLT_LEAF_VEC_I || rt.aux_class[q] == AMLT_LEAF_MAT_IJ)
            s += "        c.v[" + Q + "] = ldg_elem<T>(p.gaux[" + Q + "], i * p.gaux_si[" + Q +
                 "] + j * p.gaux_sj[" + Q + "]);\n";
    }
    s += "        (void)p; (void)i; (void)j;\n        return c;\n    }\n";
    s += "    __device__ static __forceinline__ T term(T a, T b, const Col& c) {\n";
    s += "        (void)a; (void)b; (void)c;\n        return " + rt.expr + ";\n    }\n";
    s += "    __device__ static __forceinline__ void step(Acc* acc, T a, T b, const Col& c) {\n";
    s += "        acc[0] = add_rn(acc[0], term(a, b, c));\n    }\n";
    s += "    __device__ static __forceinline__ T finish(const Acc* acc, const Col&, int64_t) {\n";
    s += "        return acc[0];\n    }\n};\n}  // namespace amltk\n";
    return s;
}

const JitBody& jit_body(const RecognizedTask& rt, int dtype, bool load) {
    Cache& C = cache();
    std::lock_guard<std::mutex> lock(C.m);
    const std::string key = key_of(rt, dtype);
    auto it = C.bodies.find(key);
    if (it != C.bodies.end() && (it->second.loaded || !load)) return it->second;

    const bool tout = has_at(rt);
    const Shape* shapes = dtype == AMLT_F64 ? kShapesF64 : kShapesF32;
    const int nshapes = kNumShapes;
    std::vector<std::string> exprs;
    for (int i = 0; i < nshapes; ++i) exprs.push_back(tile_name_expr(shapes[i], dtype, tout));
    exprs.push_back(std::string("amltk::mmlt_assign_kernel<amltk::BodyGen, ") + ctype(dtype) + ">");
    exprs.push_back(std::string("amltk::mmlt_naive_body_kernel<amltk::BodyGen, ") + ctype(dtype) + ">");

    // ---- compile (NVRTC, sm_100a) unless an earlier dry compile exists
    std::vector<char> cubin;
    std::vector<std::string> lowered(exprs.size());
    const auto t0 = std::chrono::steady_clock::now();
    const std::string src = jit_source(rt, dtype);
    const std::string disk = disk_cache_path(src);
    if (it != C.bodies.end()) {
        cubin = it->second.cubin;
        lowered = it->second.lowered;
    } else if (!disk.empty() && disk_cache_read(disk, exprs.size(), &cubin, &lowered)) {
        // compiled by an earlier process
    } else {
        const Nvrtc& N = nvrtc();
        nvrtcProgram prog = nullptr;
        if (N.create(&prog, src.c_str(), "amlt_generated_body.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS)
            throw TaskError(AMLT_ERR_ENGINE, "nvrtcCreateProgram failed");
        for (const auto& e : exprs) N.add_name(prog, e.c_str());
        const char* opts[] = {"--gpu-architecture=sm_100a", "--std=c++17", "-lineinfo",
                              "--fmad=false"};
        const nvrtcResult r = N.compile(prog, 4, opts);
        if (r != NVRTC_SUCCESS) {
            size_t ls = 0;
            N.log_size(prog, &ls);
            std::string log(ls, '\0');
            if (ls) N.log(prog, &log[0]);
            N.destroy(&prog);
            throw TaskError(AMLT_ERR_ENGINE, std::string("NVRTC failed to compile the generated body (") +
                                                 N.error(r) + "):\n" + log.substr(0, 4000));
        }
        size_t n = 0;
        N.cubin_size(prog, &n);
        cubin.resize(n);
        N.cubin(prog, cubin.data());
        for (size_t i = 0; i < exprs.size(); ++i) {
            const char* ln = nullptr;
            N.lowered(prog, exprs[i].c_str(), &ln);
            lowered[i] = ln ? ln : "";
        }
        N.destroy(&prog);
        if (!disk.empty()) disk_cache_write(disk, cubin, lowered);
    }
    const double secs =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

    // ---- load (device contexts)
    std::vector<const void*> funcs(exprs.size(), nullptr);
    if (load) {
        cudaLibrary_t lib = nullptr;
        cudaError_t e = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
        if (e != cudaSuccess)
            throw TaskError(AMLT_ERR_CUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
        for (size_t i = 0; i < exprs.size(); ++i) {
            cudaKernel_t k = nullptr;
            e = cudaLibraryGetKernel(&k, lib, lowered[i].c_str());
            if (e != cudaSuccess)
                throw TaskError(AMLT_ERR_CUDA, "cudaLibraryGetKernel(" + exprs[i] + "): " + cudaGetErrorString(e));
            funcs[i] = reinterpret_cast<const void*>(k);
        }
    }

    // ---- register (or complete an earlier dry registration)
    std::lock_guard<std::mutex> rlock(registry_mutex());
    Registry& reg = registry_mut();
    const int es = dtype == AMLT_F64 ? 8 : 4;
    JitBody* jb = nullptr;
    if (it != C.bodies.end()) {
        jb = &it->second;
    } else {
        jb = &C.bodies[key];
        jb->key = key;
        jb->dtype = dtype;
        jb->has_at = tout;
        for (int i = 0; i < nshapes; ++i) {
            const Shape& sh = shapes[i];
            VariantDesc v;
            v.body = AMLT_BODY_GENERIC;
            v.dtype = dtype;
            v.bm = sh.tm * sh.wr;
            v.bn = 32 * sh.tn * sh.wc;
            v.bk = sh.bk;
            v.tm = sh.tm;
            v.tn = sh.tn;
            v.threads = 32 * sh.wr * sh.wc;
            v.stages = sh.stages;
            v.smem = sh.stages * (v.bm * sh.bk + sh.bk * v.bn) * es + 128;
            v.minb = minb_of(sh, tout);
            v.vec = (sh.load & kTma) != 0;
            v.tout = tout;
            v.r_overwrite = true;  // the tile kernel, compiled by NVRTC
            C.names.push_back(std::string(sh.name) + (tout ? "_ti" : ""));
            v.name = C.names.back().c_str();
            v.func = nullptr;
            v.launch = nullptr;
            reg.variants.push_back(v);
            jb->variants.push_back(static_cast<int>(reg.variants.size()) - 1);
        }
        BodyAux a;
        a.body = AMLT_BODY_GENERIC;
        a.dtype = dtype;
        for (const auto& fixed : reg.aux)  // dtype-only helpers (split-K reduce, packing)
            if (fixed.body == AMLT_BODY_GEMM && fixed.dtype == dtype) {
                a.reduce = fixed.reduce;
                a.reduce_func = fixed.reduce_func;
                a.pack = fixed.pack;
                a.pack_func = fixed.pack_func;
            }
        reg.aux.push_back(a);
        jb->aux = &reg.aux.back();
    }
    if (jb->cubin.empty()) {
        jb->compile_seconds = secs;
        jb->cubin = cubin;
        jb->lowered = lowered;
    }
    if (load) {
        for (int i = 0; i < nshapes; ++i) {
            VariantDesc& v = reg.variants[static_cast<size_t>(jb->variants[static_cast<size_t>(i)])];
            v.func = funcs[static_cast<size_t>(i)];
            cudaError_t e = cudaFuncSetAttribute(v.func, cudaFuncAttributeMaxDynamicSharedMemorySize, v.smem);
            if (e != cudaSuccess)
                throw TaskError(AMLT_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        }
        BodyAux& a = const_cast<BodyAux&>(*jb->aux);
        a.assign_func = funcs[static_cast<size_t>(nshapes)];
        a.naive_func = funcs[static_cast<size_t>(nshapes) + 1];
        jb->loaded = true;
    }
    return *jb;
}

}  // namespace amltk
