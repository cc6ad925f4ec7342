// lego_runtime.cu -- C ABI of liblego_b200.so (include/lego_b200.h).
//
// Host side of the backend: NVRTC kernel JIT (dlopen'ed, so the library
// also loads on GPU-less machines), program loading through the CUDA driver
// API (dlopen'ed libcuda.so.1), and the stream-ordered launches of the
// generated layout kernels.  Fixed kernels (softmax, wavefront, GEMM) live
// in their own translation units and use the CUDA runtime directly.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/lego_b200.h"
#include "lego_common.h"

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_error;

lego_status lego_fail(lego_status code, const char* fmt, ...) {
    char buf[2048];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_error = buf;
    return code;
}

extern "C" const char* lego_last_error(void) { return g_error.c_str(); }
extern "C" int32_t lego_abi_version(void) { return LEGO_ABI_VERSION; }
extern "C" void lego_free(void* p) { free(p); }

// ---------------------------------------------------------------------------
// dynamically loaded NVRTC and driver API
// ---------------------------------------------------------------------------
typedef int nvrtcResult_t;
typedef struct _nvrtcProgram* nvrtcProgram_t;
typedef int CUresult_t;
typedef struct CUmod_st* CUmodule_t;
typedef struct CUfunc_st* CUfunction_t;

struct Nvrtc {
    void* h = nullptr;
    nvrtcResult_t (*create)(nvrtcProgram_t*, const char*, const char*, int, const char* const*,
                            const char* const*) = nullptr;
    nvrtcResult_t (*compile)(nvrtcProgram_t, int, const char* const*) = nullptr;
    nvrtcResult_t (*log_size)(nvrtcProgram_t, size_t*) = nullptr;
    nvrtcResult_t (*get_log)(nvrtcProgram_t, char*) = nullptr;
    nvrtcResult_t (*cubin_size)(nvrtcProgram_t, size_t*) = nullptr;
    nvrtcResult_t (*get_cubin)(nvrtcProgram_t, char*) = nullptr;
    nvrtcResult_t (*destroy)(nvrtcProgram_t*) = nullptr;
    const char* (*err)(nvrtcResult_t) = nullptr;
};

struct Driver {
    void* h = nullptr;
    CUresult_t (*load)(CUmodule_t*, const void*) = nullptr;
    CUresult_t (*unload)(CUmodule_t) = nullptr;
    CUresult_t (*get_fn)(CUfunction_t*, CUmodule_t, const char*) = nullptr;
    CUresult_t (*launch)(CUfunction_t, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                         unsigned, void*, void**, void**) = nullptr;
    CUresult_t (*err)(CUresult_t, const char**) = nullptr;
    CUresult_t (*set_attr)(CUfunction_t, int, int) = nullptr;
};

static std::mutex g_dl_mutex;
static Nvrtc g_nvrtc;
static Driver g_drv;

template <typename F>
static bool sym(void* h, const char* name, F& out) {
    out = reinterpret_cast<F>(dlsym(h, name));
    return out != nullptr;
}

static lego_status load_nvrtc() {
    std::lock_guard<std::mutex> lk(g_dl_mutex);
    if (g_nvrtc.h) return LEGO_OK;
    const char* names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so",
                           "/usr/local/cuda/lib64/libnvrtc.so"};
    void* h = nullptr;
    for (const char* n : names)
        if ((h = dlopen(n, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return lego_fail(LEGO_E_NVRTC, "cannot dlopen libnvrtc: %s", dlerror());
    Nvrtc n;
    n.h = h;
    bool ok = sym(h, "nvrtcCreateProgram", n.create) && sym(h, "nvrtcCompileProgram", n.compile) &&
              sym(h, "nvrtcGetProgramLogSize", n.log_size) && sym(h, "nvrtcGetProgramLog", n.get_log) &&
              sym(h, "nvrtcGetCUBINSize", n.cubin_size) && sym(h, "nvrtcGetCUBIN", n.get_cubin) &&
              sym(h, "nvrtcDestroyProgram", n.destroy) && sym(h, "nvrtcGetErrorString", n.err);
    if (!ok) return lego_fail(LEGO_E_NVRTC, "libnvrtc lacks a required symbol");
    g_nvrtc = n;
    return LEGO_OK;
}

static lego_status load_driver() {
    std::lock_guard<std::mutex> lk(g_dl_mutex);
    if (g_drv.h) return LEGO_OK;
    void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_LOCAL);
    if (!h) return lego_fail(LEGO_E_CUDA, "cannot dlopen libcuda.so.1: %s", dlerror());
    Driver d;
    d.h = h;
    bool ok = sym(h, "cuModuleLoadData", d.load) && sym(h, "cuModuleUnload", d.unload) &&
              sym(h, "cuModuleGetFunction", d.get_fn) && sym(h, "cuLaunchKernel", d.launch) &&
              sym(h, "cuGetErrorString", d.err) && sym(h, "cuFuncSetAttribute", d.set_attr);
    if (!ok) return lego_fail(LEGO_E_CUDA, "libcuda lacks a required symbol");
    g_drv = d;
    return LEGO_OK;
}

static lego_status drv_check(CUresult_t rc, const char* what) {
    if (rc == 0) return LEGO_OK;
    const char* s = "unknown";
    if (g_drv.err) g_drv.err(rc, &s);
    return lego_fail(LEGO_E_CUDA, "%s failed: %s (%d)", what, s, rc);
}

lego_status lego_cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LEGO_OK;
    return lego_fail(LEGO_E_CUDA, "%s failed: %s", what, cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// device info
// ---------------------------------------------------------------------------
extern "C" lego_status lego_device_info(int32_t device, int32_t* sm_count, int64_t* l2_bytes,
                                        int32_t* cc_major, int32_t* cc_minor) {
    cudaDeviceProp p;
    lego_status s = lego_cuda_check(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
    if (s) return s;
    if (sm_count) *sm_count = p.multiProcessorCount;
    if (l2_bytes) *l2_bytes = p.l2CacheSize;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    return LEGO_OK;
}

// ---------------------------------------------------------------------------
// NVRTC
// ---------------------------------------------------------------------------
extern "C" lego_status lego_nvrtc_compile(const char* source, size_t source_len, const char* arch,
                                          void** cubin, size_t* cubin_len, char* log,
                                          size_t log_cap) {
    if (!source || !cubin || !cubin_len) return lego_fail(LEGO_E_ARG, "null argument");
    lego_status s = load_nvrtc();
    if (s) return s;
    std::string src(source, source_len);
    std::string arch_opt = std::string("--gpu-architecture=") + (arch && *arch ? arch : "sm_100a");
    const char* opts[] = {arch_opt.c_str(), "--std=c++17", "-lineinfo", "-w"};
    nvrtcProgram_t prog = nullptr;
    nvrtcResult_t rc = g_nvrtc.create(&prog, src.c_str(), "lego_program.cu", 0, nullptr, nullptr);
    if (rc) return lego_fail(LEGO_E_NVRTC, "nvrtcCreateProgram: %s", g_nvrtc.err(rc));
    rc = g_nvrtc.compile(prog, 4, opts);
    size_t lsz = 0;
    g_nvrtc.log_size(prog, &lsz);
    std::string lg(lsz, '\0');
    if (lsz) g_nvrtc.get_log(prog, &lg[0]);
    if (log && log_cap) {
        size_t n = lg.size() < log_cap - 1 ? lg.size() : log_cap - 1;
        memcpy(log, lg.data(), n);
        log[n] = 0;
    }
    if (rc) {
        g_nvrtc.destroy(&prog);
        return lego_fail(LEGO_E_NVRTC, "nvrtcCompileProgram: %s\n%s", g_nvrtc.err(rc), lg.c_str());
    }
    size_t n = 0;
    g_nvrtc.cubin_size(prog, &n);
    void* buf = malloc(n);
    if (!buf) {
        g_nvrtc.destroy(&prog);
        return lego_fail(LEGO_E_ARG, "out of host memory");
    }
    g_nvrtc.get_cubin(prog, static_cast<char*>(buf));
    g_nvrtc.destroy(&prog);
    *cubin = buf;
    *cubin_len = n;
    return LEGO_OK;
}

// ---------------------------------------------------------------------------
// programs
// ---------------------------------------------------------------------------
struct lego_program_s {
    lego_program_info info;
    CUmodule_t mod = nullptr;
    CUfunction_t remap = nullptr, remap_fill = nullptr;
    CUfunction_t apply32 = nullptr, apply64 = nullptr, inv32 = nullptr, inv64 = nullptr;
    CUfunction_t hist = nullptr, hist_check = nullptr;
    CUfunction_t nw_tiles = nullptr, nw_borders = nullptr;
    CUfunction_t sm_rows = nullptr, sm_offsets = nullptr;
};

extern "C" lego_status lego_program_load(const void* cubin, size_t cubin_len,
                                         const lego_program_info* info, lego_program* out) {
    (void)cubin_len;
    if (!cubin || !info || !out) return lego_fail(LEGO_E_ARG, "null argument");
    lego_status s = load_driver();
    if (s) return s;
    // make the device's primary context current on this thread (PyTorch uses it too)
    int dev = 0;
    if ((s = lego_cuda_check(cudaGetDevice(&dev), "cudaGetDevice"))) return s;
    if ((s = lego_cuda_check(cudaFree(nullptr), "cudaFree(0)"))) return s;
    auto* p = new lego_program_s();
    p->info = *info;
    if ((s = drv_check(g_drv.load(&p->mod, cubin), "cuModuleLoadData"))) {
        delete p;
        return s;
    }
    if (info->kind == LEGO_PROG_INDEX_MAP) {
        bool ok = !g_drv.get_fn(&p->apply32, p->mod, "lego_apply_map_i32") &&
                  !g_drv.get_fn(&p->apply64, p->mod, "lego_apply_map_i64") &&
                  !g_drv.get_fn(&p->inv32, p->mod, "lego_inv_map_i32") &&
                  !g_drv.get_fn(&p->inv64, p->mod, "lego_inv_map_i64") &&
                  !g_drv.get_fn(&p->hist, p->mod, "lego_hist") &&
                  !g_drv.get_fn(&p->hist_check, p->mod, "lego_hist_check");
        if (!ok) {
            g_drv.unload(p->mod);
            delete p;
            return lego_fail(LEGO_E_ARG, "index-map program lacks its kernels");
        }
    } else if (info->kind == LEGO_PROG_SOFTMAX) {
        bool ok = !g_drv.get_fn(&p->sm_rows, p->mod, "lego_softmax_rows") &&
                  !g_drv.get_fn(&p->sm_offsets, p->mod, "lego_softmax_offsets");
        if (!ok) {
            g_drv.unload(p->mod);
            delete p;
            return lego_fail(LEGO_E_ARG, "softmax program lacks its kernels");
        }
    } else if (info->kind == LEGO_PROG_NW) {
        if (info->smem_bytes < lego_nw_smem_bytes()) {
            g_drv.unload(p->mod);
            delete p;
            return lego_fail(LEGO_E_ARG, "NW program shared memory %d != the library's %d", info->smem_bytes,
                             lego_nw_smem_bytes());
        }
        bool ok = !g_drv.get_fn(&p->nw_tiles, p->mod, "lego_nw_tiles") &&
                  !g_drv.get_fn(&p->nw_borders, p->mod, "lego_nw_borders");
        if (!ok) {
            g_drv.unload(p->mod);
            delete p;
            return lego_fail(LEGO_E_ARG, "NW program lacks its kernels");
        }
        if ((s = drv_check(g_drv.set_attr(p->nw_tiles, 8 /*MAX_DYNAMIC_SHARED_SIZE_BYTES*/, info->smem_bytes),
                           "cuFuncSetAttribute(nw)"))) {
            g_drv.unload(p->mod);
            delete p;
            return s;
        }
    } else {
        if ((s = drv_check(g_drv.get_fn(&p->remap, p->mod, "lego_remap"), "cuModuleGetFunction(lego_remap)"))) {
            g_drv.unload(p->mod);
            delete p;
            return s;
        }
        if (info->smem_bytes > 48 * 1024)
            g_drv.set_attr(p->remap, 8 /*CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES*/, info->smem_bytes);
        if ((info->reserved & (LEGO_FILL_FUSED | LEGO_FILL_PASS)) &&
            (s = drv_check(g_drv.get_fn(&p->remap_fill, p->mod, "lego_remap_fill"),
                           "cuModuleGetFunction(lego_remap_fill)"))) {
            g_drv.unload(p->mod);
            delete p;
            return s;
        }
    }
    *out = p;
    return LEGO_OK;
}

extern "C" void lego_program_release(lego_program p) {
    if (!p) return;
    if (p->mod && g_drv.unload) g_drv.unload(p->mod);
    delete p;
}

static lego_status launch(CUfunction_t fn, unsigned gx, unsigned gy, unsigned block, unsigned smem,
                          void* stream, void** args) {
    return drv_check(g_drv.launch(fn, gx, gy, 1, block, 1, 1, smem, stream, args, nullptr),
                     "cuLaunchKernel");
}

static unsigned map_grid(int64_t count) {
    int64_t g = (count + 255) / 256;
    const int64_t cap = 148 * 64;   // grid-stride beyond ~64 CTAs per SM
    if (g > cap) g = cap;
    return (unsigned)(g < 1 ? 1 : g);
}

static lego_status index_map(lego_program p, int which, void* out, int32_t out_bytes, int64_t first,
                             int64_t count, void* stream) {
    if (!p || p->info.kind != LEGO_PROG_INDEX_MAP)
        return lego_fail(LEGO_E_ARG, "program is not an index-map program");
    if (out_bytes != 4 && out_bytes != 8) return lego_fail(LEGO_E_ARG, "out_bytes must be 4 or 8");
    if (count < 0 || first < 0) return lego_fail(LEGO_E_BOUNDS, "negative range");
    if (count == 0) return LEGO_OK;
    if (!out) return lego_fail(LEGO_E_ARG, "null output");
    CUfunction_t fn = which == 0 ? (out_bytes == 4 ? p->apply32 : p->apply64)
                                 : (out_bytes == 4 ? p->inv32 : p->inv64);
    void* args[] = {&out, &first, &count};
    return launch(fn, map_grid(count), 1, 256, 0, stream, args);
}

extern "C" lego_status lego_apply_map(lego_program p, void* out, int32_t out_bytes, int64_t first,
                                      int64_t count, void* stream) {
    if (p && first + count > p->info.n)
        return lego_fail(LEGO_E_BOUNDS, "range [%lld, %lld) outside the logical space of %lld",
                         (long long)first, (long long)(first + count), (long long)p->info.n);
    return index_map(p, 0, out, out_bytes, first, count, stream);
}

extern "C" lego_status lego_inv_map(lego_program p, void* out, int32_t out_bytes, int64_t first,
                                    int64_t count, void* stream) {
    if (p && first + count > p->info.units)
        return lego_fail(LEGO_E_BOUNDS, "range [%lld, %lld) outside the physical space of %lld",
                         (long long)first, (long long)(first + count), (long long)p->info.units);
    return index_map(p, 1, out, out_bytes, first, count, stream);
}

static lego_status check_hits(lego_program p, uint32_t* hist, int64_t* violations, int at_most_once,
                              void* stream) {
    if (!p || p->info.kind != LEGO_PROG_INDEX_MAP)
        return lego_fail(LEGO_E_ARG, "program is not an index-map program");
    if (!hist || !violations) return lego_fail(LEGO_E_ARG, "null argument");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t n_out = p->info.units;   // physical size
    int64_t count = p->info.n;       // logical size
    unsigned long long* bad = nullptr;
    lego_status s;
    if ((s = lego_cuda_check(cudaMallocAsync((void**)&bad, sizeof(unsigned long long), st), "cudaMallocAsync")))
        return s;
    cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st);
    cudaMemsetAsync(hist, 0, sizeof(uint32_t) * (size_t)n_out, st);
    void* a1[] = {&hist, &count, &n_out, &bad};
    if ((s = launch(p->hist, map_grid(count), 1, 256, 0, stream, a1))) return s;
    void* a2[] = {&hist, &n_out, &bad, &at_most_once};
    if ((s = launch(p->hist_check, map_grid(n_out), 1, 256, 0, stream, a2))) return s;
    unsigned long long host = 0;
    cudaMemcpyAsync(&host, bad, sizeof host, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(bad, st);
    if ((s = lego_cuda_check(cudaStreamSynchronize(st), "cudaStreamSynchronize"))) return s;
    *violations = (int64_t)host;
    return LEGO_OK;
}

extern "C" lego_status lego_check_bijective(lego_program p, uint32_t* hist, int64_t* violations,
                                            void* stream) {
    return check_hits(p, hist, violations, 0, stream);
}

extern "C" lego_status lego_check_injective(lego_program p, uint32_t* hist, int64_t* violations,
                                            void* stream) {
    return check_hits(p, hist, violations, 1, stream);
}

// ---------------------------------------------------------------------------
// user modules: kernels instantiated from LEGO templates (template.instantiate
// with [target] cuda), compiled by lego_nvrtc_compile and launched by name
// ---------------------------------------------------------------------------
struct lego_module_s {
    CUmodule_t mod = nullptr;
};

extern "C" lego_status lego_module_load(const void* cubin, size_t cubin_len, lego_module* out) {
    (void)cubin_len;
    if (!cubin || !out) return lego_fail(LEGO_E_ARG, "null argument");
    lego_status s = load_driver();
    if (s) return s;
    if ((s = lego_cuda_check(cudaFree(nullptr), "cudaFree(0)"))) return s;
    auto* m = new lego_module_s();
    if ((s = drv_check(g_drv.load(&m->mod, cubin), "cuModuleLoadData"))) {
        delete m;
        return s;
    }
    *out = m;
    return LEGO_OK;
}

extern "C" void lego_module_release(lego_module m) {
    if (!m) return;
    if (m->mod && g_drv.unload) g_drv.unload(m->mod);
    delete m;
}

extern "C" lego_status lego_module_launch(lego_module m, const char* kernel, uint32_t gx, uint32_t gy, uint32_t gz,
                                          uint32_t bx, uint32_t by, uint32_t bz, uint32_t smem, void** args,
                                          void* stream) {
    if (!m || !kernel) return lego_fail(LEGO_E_ARG, "null argument");
    CUfunction_t fn = nullptr;
    lego_status s = drv_check(g_drv.get_fn(&fn, m->mod, kernel), "cuModuleGetFunction");
    if (s) return s;
    if (smem > 48 * 1024 && (s = drv_check(g_drv.set_attr(fn, 8, (int)smem), "cuFuncSetAttribute"))) return s;
    return drv_check(g_drv.launch(fn, gx, gy, gz, bx, by, bz, smem, stream, args, nullptr), "cuLaunchKernel");
}

extern "C" lego_status lego_softmax_run(lego_program p, const float* x, float* y, int64_t rows, int64_t cols,
                                        void* stream) {
    if (!p || p->info.kind != LEGO_PROG_SOFTMAX) return lego_fail(LEGO_E_ARG, "program is not a softmax program");
    if (cols != p->info.n)
        return lego_fail(LEGO_E_SHAPE, "program was built for %lld columns, called with %lld",
                         (long long)p->info.n, (long long)cols);
    if (rows < 0 || rows > p->info.units || rows > 0x7fffffffLL)
        return lego_fail(LEGO_E_SHAPE, "rows %lld outside the program's layout (%lld)", (long long)rows,
                         (long long)p->info.units);
    if (rows == 0) return LEGO_OK;
    if (!x || !y) return lego_fail(LEGO_E_ARG, "null buffer");
    if (((uintptr_t)x | (uintptr_t)y) & 15) return lego_fail(LEGO_E_ARG, "buffers must be 16-byte aligned");
    void* args[] = {&x, &y};
    return launch(p->sm_rows, (unsigned)rows, 1, (unsigned)p->info.block, 0, stream, args);
}

extern "C" lego_status lego_softmax_offsets(lego_program p, int64_t* out, int64_t rows, void* stream) {
    if (!p || p->info.kind != LEGO_PROG_SOFTMAX) return lego_fail(LEGO_E_ARG, "program is not a softmax program");
    if (rows < 0 || rows > p->info.units || rows > 0x7fffffffLL) return lego_fail(LEGO_E_SHAPE, "bad rows");
    if (rows == 0) return LEGO_OK;
    if (!out) return lego_fail(LEGO_E_ARG, "null buffer");
    void* args[] = {&out};
    return launch(p->sm_offsets, (unsigned)rows, 1, (unsigned)p->info.block, 0, stream, args);
}

extern "C" lego_status lego_nw_run(lego_program p, const int32_t* sim, int32_t* score, int64_t n,
                                   int32_t penalty, int64_t batch, void* stream) {
    if (!p || p->info.kind != LEGO_PROG_NW) return lego_fail(LEGO_E_ARG, "program is not an NW program");
    if (n != p->info.n)
        return lego_fail(LEGO_E_SHAPE, "program was built for n = %lld, called with n = %lld",
                         (long long)p->info.n, (long long)n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    NwPlan pl;
    lego_status s = lego_nw_prepare(sim, score, n, penalty, batch, p->info.units, p->info.reserved & 1, st, &pl);
    if (s || batch == 0) return s;
    long long nn = n, bb = batch;
    int pp = penalty;
    void* a1[] = {&score, &nn, &pp, &bb};
    if ((s = launch(p->nw_borders, pl.border_ctas, 1, 256, 0, stream, a1))) return s;
    if (n == 0) return LEGO_OK;
    int ni = (int)n;
    void* a2[] = {&sim, &score, &ni, &pp, &pl.H, &pl.nr, &pl.nc, &pl.total, &pl.ticket, &pl.bnd, &pl.top};
    return launch(p->nw_tiles, pl.ctas, 1, 128, (unsigned)p->info.smem_bytes, stream, a2);
}

static lego_status remap_args(lego_program p, const void* src, void* dst, int64_t batch, int64_t src_stride,
                              int64_t dst_stride);

extern "C" lego_status lego_remap_fill(lego_program p, const void* src, void* dst, int64_t batch,
                                       int64_t src_stride, int64_t dst_stride, const void* fill, void* stream) {
    if (!p || !(p->info.reserved & (LEGO_FILL_FUSED | LEGO_FILL_PASS)))
        return lego_fail(LEGO_E_ARG, "program was not built with a fill mode");
    if (!fill) return lego_fail(LEGO_E_ARG, "null fill value");
    lego_status s = remap_args(p, src, dst, batch, src_stride, dst_stride);
    if (s || batch == 0) return s;
    unsigned long long bits = 0;
    memcpy(&bits, fill, (size_t)p->info.elem_bytes);
    void* args[] = {&src, &dst, &src_stride, &dst_stride, &bits};
    if (p->info.reserved & LEGO_FILL_FUSED)
        return launch(p->remap_fill, (unsigned)p->info.units, (unsigned)batch, (unsigned)p->info.block, 0, stream,
                      args);
    if ((s = launch(p->remap_fill, 148 * 4, (unsigned)batch, 256, 0, stream, args))) return s;
    void* a2[] = {&src, &dst, &src_stride, &dst_stride};
    return launch(p->remap, (unsigned)p->info.units, (unsigned)batch, (unsigned)p->info.block,
                  (unsigned)p->info.smem_bytes, stream, a2);
}

extern "C" lego_status lego_remap(lego_program p, const void* src, void* dst, int64_t batch,
                                  int64_t src_stride, int64_t dst_stride, void* stream) {
    lego_status s = remap_args(p, src, dst, batch, src_stride, dst_stride);
    if (s || batch == 0) return s;
    if (p->info.reserved & LEGO_FILL_FUSED)
        return lego_fail(LEGO_E_ARG, "fused fill program: call lego_remap_fill");
    void* args[] = {&src, &dst, &src_stride, &dst_stride};
    return launch(p->remap, (unsigned)p->info.units, (unsigned)batch, (unsigned)p->info.block,
                  (unsigned)p->info.smem_bytes, stream, args);
}

static lego_status remap_args(lego_program p, const void* src, void* dst, int64_t batch, int64_t src_stride,
                              int64_t dst_stride) {
    if (!p || p->info.kind == LEGO_PROG_INDEX_MAP)
        return lego_fail(LEGO_E_ARG, "program is not a remap program");
    if (batch < 0) return lego_fail(LEGO_E_ARG, "negative batch");
    if (batch == 0) return LEGO_OK;
    if (!src || !dst) return lego_fail(LEGO_E_ARG, "null buffer");
    if (batch > 65535) return lego_fail(LEGO_E_ARG, "batch above 65535: split the call");
    const int e = p->info.elem_bytes;
    const bool src_vec = !(p->info.reserved & LEGO_ALIGN_SRC_FREE);
    const bool dst_vec = !(p->info.reserved & LEGO_ALIGN_DST_FREE);
    const uintptr_t amask = (uintptr_t)(e < 16 ? e - 1 : 15);
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & amask)
        return lego_fail(LEGO_E_ARG, "buffers must be element-aligned");
    if ((src_vec && (reinterpret_cast<uintptr_t>(src) & 15)) || (dst_vec && (reinterpret_cast<uintptr_t>(dst) & 15)))
        return lego_fail(LEGO_E_ARG, "buffers must be 16-byte aligned");
    if (batch > 1 && ((src_vec && ((src_stride * e) & 15)) || (dst_vec && ((dst_stride * e) & 15))))
        return lego_fail(LEGO_E_ARG, "batch strides must be multiples of 16 bytes");
    return LEGO_OK;
}
