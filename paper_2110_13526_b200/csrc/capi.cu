// capi.cu -- error reporting, launch accounting and the reference-signature entry
// points (drop-ins for the Numba kernels of operator.py:190-233).
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <vector>

#include "cbct_internal.cuh"

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

int cbct_fail(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int cbct_fail_cuda(cudaError_t e, const char* what) {
    snprintf(g_err, sizeof(g_err), "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return (int)e;
}

void cbct_count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

extern "C" const char* cbct_last_error(void) { return g_err; }
extern "C" int cbct_version(void) { return 100; }
extern "C" int64_t cbct_launch_count(void) { return g_launches.load(); }

// ---------------------------------------------------------------------------
// Reference-signature entry points: host fp64 in the reference layouts.
// A one-entry plan cache keyed on the full geometry avoids rebuilding the
// tables when a caller (e.g. a solver loop through this ABI) repeats a geometry.
namespace {
struct RefCache {
    std::mutex mu;
    std::vector<double> key;
    cbct_plan* plan = nullptr;
} g_cache;

int get_plan(const double* srcs, const double* det00, const double* ustep, const double* vstep, int64_t V,
             int64_t nu, int64_t nv, double lo0, double lo1, double lo2, double p0, double p1, double p2,
             int64_t n0, int64_t n1, int64_t n2, cbct_plan** out) {
    std::vector<double> key = {(double)V, (double)nu, (double)nv, lo0, lo1, lo2, p0, p1, p2,
                               (double)n0, (double)n1, (double)n2};
    key.insert(key.end(), srcs, srcs + 3 * V);
    key.insert(key.end(), det00, det00 + 3 * V);
    key.insert(key.end(), ustep, ustep + 3 * V);
    key.insert(key.end(), vstep, vstep + 3 * V);
    if (g_cache.plan && g_cache.key.size() == key.size() &&
        memcmp(g_cache.key.data(), key.data(), key.size() * sizeof(double)) == 0) {
        *out = g_cache.plan;
        return 0;
    }
    cbct_geometry g;
    g.nx = n0; g.ny = n1; g.nz = n2;
    g.lo[0] = lo0; g.lo[1] = lo1; g.lo[2] = lo2;
    g.pitch[0] = p0; g.pitch[1] = p1; g.pitch[2] = p2;
    g.nu = nu; g.nv = nv; g.n_views = V;
    g.srcs = srcs; g.det00 = det00; g.ustep = ustep; g.vstep = vstep;
    cbct_plan* p = nullptr;
    int rc = cbct_plan_create(&p, &g, nullptr);
    if (rc) return rc;
    if (g_cache.plan) cbct_plan_destroy(g_cache.plan);
    g_cache.plan = p;
    g_cache.key.swap(key);
    *out = p;
    return 0;
}

struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { if (p) cudaFree(p); }
};
}  // namespace

extern "C" int cbct_ref_project(const double* vol, double* out, const double* srcs, const double* det00,
                                const double* ustep, const double* vstep, int64_t V, int64_t nu, int64_t nv,
                                double lo0, double lo1, double lo2, double p0, double p1, double p2, int64_t n0,
                                int64_t n1, int64_t n2) {
    if (!vol || !out) return cbct_fail(CBCT_E_ARG, "cbct_ref_project: null argument");
    std::lock_guard<std::mutex> lk(g_cache.mu);
    cbct_plan* p = nullptr;
    int rc = get_plan(srcs, det00, ustep, vstep, V, nu, nv, lo0, lo1, lo2, p0, p1, p2, n0, n1, n2, &p);
    if (rc) return rc;
    const int64_t n = n0 * n1 * n2, m = V * nu * nv;
    DevBuf h_in, d_in, d_vol, d_proj, d_out;
    CBCT_CHECK(cudaMalloc(&d_in.p, n * sizeof(double)));
    CBCT_CHECK(cudaMalloc(&d_vol.p, p->vol_elems * sizeof(float)));
    CBCT_CHECK(cudaMalloc(&d_proj.p, m * sizeof(float)));
    CBCT_CHECK(cudaMalloc(&d_out.p, m * sizeof(double)));
    CBCT_CHECK(cudaMemcpy(d_in.p, vol, n * sizeof(double), cudaMemcpyHostToDevice));
    if ((rc = cbct_volume_to_internal(p, d_in.p, 1, (float*)d_vol.p, nullptr))) return rc;
    if ((rc = cbct_project(p, (const float*)d_vol.p, (float*)d_proj.p, nullptr, nullptr))) return rc;
    if ((rc = cbct_proj_from_internal(p, (const float*)d_proj.p, d_out.p, 1, nullptr))) return rc;
    CBCT_CHECK(cudaMemcpy(out, d_out.p, m * sizeof(double), cudaMemcpyDeviceToHost));
    return 0;
}

extern "C" int cbct_ref_backproject(const double* proj, double* out, const double* srcs, const double* det00,
                                    const double* ustep, const double* vstep, int64_t V, int64_t nu, int64_t nv,
                                    double lo0, double lo1, double lo2, double p0, double p1, double p2, int64_t n0,
                                    int64_t n1, int64_t n2, int64_t n_workers, int mode) {
    (void)n_workers;  // the gather is deterministic for any worker count
    if (!out || (mode == 1 && !proj)) return cbct_fail(CBCT_E_ARG, "cbct_ref_backproject: null argument");
    std::lock_guard<std::mutex> lk(g_cache.mu);
    cbct_plan* p = nullptr;
    int rc = get_plan(srcs, det00, ustep, vstep, V, nu, nv, lo0, lo1, lo2, p0, p1, p2, n0, n1, n2, &p);
    if (rc) return rc;
    const int64_t n = n0 * n1 * n2, m = V * nu * nv;
    DevBuf d_in, d_proj, d_scr, d_vol, d_out;
    CBCT_CHECK(cudaMalloc(&d_proj.p, m * sizeof(float)));
    cbct_plan_info info;
    cbct_plan_get_info(p, &info);
    CBCT_CHECK(cudaMalloc(&d_scr.p, info.bp_scratch_floats * sizeof(float)));
    CBCT_CHECK(cudaMalloc(&d_vol.p, p->vol_elems * sizeof(float)));
    CBCT_CHECK(cudaMalloc(&d_out.p, n * sizeof(double)));
    if (mode == 1) {
        CBCT_CHECK(cudaMalloc(&d_in.p, m * sizeof(double)));
        CBCT_CHECK(cudaMemcpy(d_in.p, proj, m * sizeof(double), cudaMemcpyHostToDevice));
        if ((rc = cbct_proj_to_internal(p, d_in.p, 1, (float*)d_proj.p, nullptr))) return rc;
    }
    if ((rc = cbct_backproject(p, (const float*)d_proj.p, (float*)d_vol.p, mode, (float*)d_scr.p, nullptr, nullptr,
                               nullptr)))
        return rc;
    if ((rc = cbct_volume_from_internal(p, (const float*)d_vol.p, d_out.p, 1, nullptr))) return rc;
    std::vector<double> tmp((size_t)n);
    CBCT_CHECK(cudaMemcpy(tmp.data(), d_out.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    for (int64_t j = 0; j < n; ++j) out[j] += tmp[(size_t)j];  // operator.py:231-233 accumulates into out
    return 0;
}
