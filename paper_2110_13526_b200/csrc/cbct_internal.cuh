// cbct_internal.cuh -- private types and helpers of libcbct.so (sm_100a).
//
// Data layout in HBM:
//   volume      [ny][nx][zs]   fp32, zs = round_up(nz + 2*CBCT_ZPAD, 4), z fastest; slices
//                              [0,ZPAD) and [ZPAD+nz, zs) are zero guards
//   projections [V][nu][nv]    fp32, detector row v fastest
//   column table (A):    per detector column c = view*nu + u, entries
//                        [col_off[c], col_off[c+1]) of {tau_end fp32, cell_base int32}
//   cell table   (A^T):  per cell (iy*nx+ix), entries [cell_off[k], cell_off[k+1])
//                        of {vu int32, tau_a fp32, tau_b fp32}
// tau = t - t_ref(column): ray parameter relative to a per-column anchor, which
// keeps fp32 interval ends accurate to ~1e-8 of the ray (hard part 1).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/cbct.h"

// NVTX range over an entry point (header-only NVTX3: a no-op unless a profiler injects itself),
// so nsys / ncu --nvtx timelines show which operator call a kernel belongs to.
struct CbctRange {
    explicit CbctRange(const char* name) { nvtxRangePushA(name); }
    ~CbctRange() { nvtxRangePop(); }
    CbctRange(const CbctRange&) = delete;
    CbctRange& operator=(const CbctRange&) = delete;
};

#define CBCT_CHECK(expr)                                       \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cbct_fail_cuda(_e, #expr); \
    } while (0)

// Checked build (make CHECKED=1 -> build-checked/libcbct_checked.so, loaded with CBCT_LIBRARY):
// device-side bounds checks on the gathers and shared-memory indexing of the hot kernels, the
// substitute for compute-sanitizer (closed on this GPU pool).  A failed check prints the
// condition and traps; the default build compiles them out.
#ifdef CBCT_CHECKED
#include <cstdio>
#define CBCT_DCHECK(cond)                                                                         \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("CBCT_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,       \
                   (int)blockIdx.x, (int)threadIdx.x, #cond);                                     \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define CBCT_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

int cbct_fail_cuda(cudaError_t e, const char* what);
int cbct_fail(int code, const char* msg);
void cbct_count_launch(int n = 1);

struct ColumnHeader {  // one detector column (view, u); fp64 facts from the plan builder
    double tmin, tmax;  // xy box clip of the column's rays (operator.py:60-100), within [0,1]
    double rxy2;        // rx^2 + ry^2
    float t_ref;        // anchor, exactly representable in fp32
    float tau_start;    // tmin - t_ref
    int32_t flat_slab;  // z slab of a flat (|rz| < 1e-12 p2) ray in this column, or INT32_MIN
    int32_t pad;
};

struct CellEntry {  // one column crossing a cell, in cell-major order
    int32_t vu;
    float tau_a, tau_b;
};

struct cbct_plan {
    // geometry (host copies)
    int64_t nx, ny, nz, zs;
    double lo[3], pitch[3];
    int64_t nu, nv, V;
    double det00z, pv;  // detector row geometry shared by all views (v_axis = +z)
    int32_t flat_v;     // index of the flat row (|w| < 1e-12 p2) or -1
    // sizes
    int64_t n_cols, n_cells, n_intervals, max_intervals, max_cell_entries;
    // shard plan (cbct_plan_create_shard): the column table holds views [own_v0, own_v1), the cell
    // table cell rows [own_r0, own_r1); the unsharded plan owns everything
    int64_t own_v0 = 0, own_v1 = 0, own_r0 = 0, own_r1 = 0;
    bool sharded = false;
    int32_t* d_pref_cols = nullptr;  // shard plan: columns with entries in the plan's cell rows (A^T prefix)
    int64_t n_pref_cols = 0;
    int64_t vol_elems, n_rays;
    size_t table_bytes;
    // device tables
    ColumnHeader* d_cols = nullptr;
    int64_t* d_col_off = nullptr;   // n_cols + 1
    float2* d_col_ent = nullptr;    // {tau_end, __int_as_float(cell_base)} n_intervals
    int64_t* d_cell_off = nullptr;  // n_cells + 1
    int32_t* d_cell_boff = nullptr;  // n_cells x (bp_vbatch + 1): entry offsets of the view batches in a cell
    int32_t bp_vbatch = 1;           // A^T launches over view batches (L2 working set)
    CellEntry* d_cell_ent = nullptr;
    double* d_srcs = nullptr;       // per-view tables of _view_tables (operator.py:262-281), [V][3] fp64
    double* d_det00 = nullptr;
    double* d_ustep = nullptr;
    double* d_vstep = nullptr;
    double* d_len64 = nullptr;      // fp64 path (f64.cu): |r| per ray, internal order; cbct_plan_enable_f64
    void* d_rayz64 = nullptr;       // fp64 path: per-ray box clip and z-walk start (f64.cu RayZ)
    void* d_rayiz64 = nullptr;      // fp64 path: per-ray entry slab and z step (int2)
    void* d_cell_t64 = nullptr;     // fp64 path: per cell entry, the column walk's t bounding the crossing
    double* d_w = nullptr;          // per-row rz (fp64), nv
    float* d_invw = nullptr;        // per-row 1/rz (fp32; +-1e30 for flat rows), nv
    // launch shapes
    int proj_threads, proj_rpt;
    int proj_tma, proj_tma_k, proj_tma_stages;  // TMA-staged projector shape
    int proj_q, proj_q_c, proj_q_zr;            // column prefix-sum projector (chunk of C cells, zero row)
    int bp_threads, bp_zpt;
    int bpg_threads, bpg_groups;  // boundary-form backprojector shape
    // sided boundary kernel (k_bp_sided): GS below + GS above groups per warp, anchored at the
    // first boundary k0 with z >= 0; usable when z_k0 == 0 exactly or one side is empty
    bool bps_ok = false;        // mode 1 runs k_bp_sided (geometry eligible and <= 10% wasted slots)
    bool bps_eligible = false;  // geometry allows k_bp_sided (mode 2 uses it whenever eligible)
    bool bps_mode2_ok = false;  // no ray's z range inside one crossing reaches a voxel height
    int bps_gs = 0, bps_threads = 0, bps_k0 = 0, bps_zero = 0;
    bool bp_boundary_ok;          // at most one ray straddles any voxel boundary per crossing
    int32_t bp_pad_lo, bp_pad_hi; // rows of the ray-prefix table below 0 / above nv (no index clamping)
    bool bp_closed_ok;            // eps = max dtau / min t small enough for the closed-form straddle
    float max_dtau;               // longest column/cell interval (ray parameter)
    int32_t proj_blocks, bp_blocks;
};

__device__ __forceinline__ int floor_to_int(double x) { return (int)floor(x); }
