/*
 * include/cbct.h -- C ABI of the B200-native cone-beam projector pair (libcbct.so).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * cbctkit 0.1.0 (/root/reference/pkg/src/cbctkit).  The reference's hot path is
 * two Numba kernels behind CbctOperator:
 *
 *   _project_kernel(vol, out, srcs, det00, ustep, vstep, nu, nv,
 *                   lo0, lo1, lo2, p0, p1, p2, n0, n1, n2)          operator.py:190-206
 *   _backproject_kernel(proj, out, srcs, det00, ustep, vstep, nu, nv,
 *                   lo0, lo1, lo2, p0, p1, p2, n0, n1, n2,
 *                   n_workers, mode)                               operator.py:209-233
 *
 * and the CGLS/LSQR/PSIRT vector updates in solvers.py:269-569.
 *
 * Two levels are exported:
 *
 *  1. Stateless reference-signature entry points (cbct_ref_project /
 *     cbct_ref_backproject): host fp64 buffers in the reference layouts
 *     (volume x-fastest (nz,ny,nx); projections u-fastest (V,nv,nu)), the same
 *     argument list as the Numba kernels.  They build (and cache) a plan, copy
 *     in, run the CUDA kernels, copy out.  This is what a ctypes/cffi binding of
 *     the reference would call in place of the Numba kernels.
 *
 *  2. The plan API used by the Python package: a cbct_plan owns the
 *     device-resident fan-beam tables of one (volume, trajectory) pair and all
 *     kernels run on caller-provided device buffers (torch-owned) in the
 *     internal layouts:
 *        volume:      [ny][nx][zs] fp32, z fastest, zs = round_up(nz + 2*CBCT_ZPAD, 4);
 *                     slices [0,ZPAD) and [ZPAD+nz, zs) are zero guards
 *        projections: [n_views][nu][nv] fp32, v (detector row) fastest
 *     Launches are asynchronous on the given stream, never allocate, and are
 *     deterministic (no atomics on data).
 *
 * Every function returns 0 on success or a positive cudaError_t / negative
 * CBCT_E* code; nothing throws across the ABI.  cbct_last_error() returns a
 * message for the last failure on the calling thread.
 */
#ifndef CBCT_H
#define CBCT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBCT_ZPAD 4 /* zero guard slices on each side of z in the internal volume layout */

enum {
    CBCT_OK = 0,
    CBCT_E_ARG = -1,       /* invalid argument */
    CBCT_E_GEOMETRY = -2,  /* geometry outside the supported family */
    CBCT_E_NOMEM = -3,     /* device allocation failed */
    CBCT_E_NODEVICE = -4,  /* no CUDA device */
};

/* Geometry of one operator, host memory.  Mirrors CbctOperator's inputs
 * (operator.py:292-314): the per-view tables are those of _view_tables
 * (operator.py:262-281), [n_views][3] fp64 each. */
typedef struct cbct_geometry {
    int64_t nx, ny, nz;        /* VolumeGeometry counts (geometry.py:44-46) */
    double lo[3];              /* VolumeGeometry.corner() (geometry.py:69-74) */
    double pitch[3];           /* voxel_size */
    int64_t nu, nv, n_views;   /* DetectorGeometry nu, nv; TrajectoryGeometry n_views */
    const double* srcs;        /* source_position per view */
    const double* det00;       /* centre of pixel (0,0) per view */
    const double* ustep;       /* pu * u_axis per view */
    const double* vstep;       /* pv * v_axis per view */
} cbct_geometry;

typedef struct cbct_plan cbct_plan;

/* Static facts about a plan (sizes of the internal layouts and of the tables). */
typedef struct cbct_plan_info {
    int64_t n_voxels;          /* nx*ny*nz */
    int64_t n_rays;            /* n_views*nu*nv */
    int64_t vol_elems;         /* padded internal volume length: ny*nx*zstride */
    int64_t zstride;           /* round_up(nz + 2*CBCT_ZPAD, 4) */
    int64_t n_columns;         /* n_views*nu detector columns */
    int64_t n_intervals;       /* column/cell intersections = nnz of the 2-D fan-beam matrix */
    int64_t max_intervals;     /* longest column list */
    int64_t max_cell_entries;  /* longest cell list */
    int64_t table_bytes;       /* device bytes held by the plan */
    int32_t proj_blocks;       /* number of fp64 partials written by cbct_project */
    int32_t bp_blocks;         /* number of fp64 partials written by cbct_backproject */
    int64_t bp_scratch_floats; /* fp32 workspace cbct_backproject needs (scratch_proj) */
    int32_t bp_fast_path;      /* 1: mode-1 A^T uses the boundary-form kernel */
    int32_t bp_closed_form;    /* 1: its straddle fraction is the closed form (no 1/rz table) */
    /* launch shapes the plan chose (appended; read-only diagnostics) */
    int32_t proj_chunk;        /* cells per chunk of the prefix-sum projector (0: another projector) */
    int32_t bp_groups;         /* boundary groups per warp of the boundary-form backprojector */
    int32_t bp_view_batches;   /* launches of one mode-1 backprojection (view batches) */
    int32_t bp_sided_gs;       /* 0: mode-1 A^T runs k_bp_boundary; g > 0: k_bp_sided with g below + g above
                                  boundary groups per warp */
} cbct_plan_info;

/* ---- plan lifecycle ------------------------------------------------------ */
/* Build the fan-beam tables on the current CUDA device (synchronous).
 * Replaces CbctOperator.__init__'s table setup (operator.py:292-301). */
int cbct_plan_create(cbct_plan** plan, const cbct_geometry* geom, void* stream);
int cbct_plan_destroy(cbct_plan* plan);
/* A plan for one rank of the sharded operator: the column table of views
 * [view0, view1) only (cbct_project_views inside that block) and the cell table of cell rows
 * [row0, row1) only (cbct_backproject_rows inside that block), so the tables shrink ~1/world.
 * Within its blocks it computes exactly what the unsharded plan computes (same tables for those
 * views / rows, same launch shapes).  No fp64 path (cbct_plan_enable_f64 refuses). */
int cbct_plan_create_shard(cbct_plan** plan, const cbct_geometry* geom, int64_t view0, int64_t view1,
                           int64_t row0, int64_t row1, void* stream);
int cbct_plan_get_info(const cbct_plan* plan, cbct_plan_info* info);

/* ---- operators on device buffers (internal layouts) ----------------------- */
/* proj = A vol  (operator.py:190-206, 316-326).  If norm2_partials != NULL, it
 * receives info.proj_blocks fp64 partial sums of proj^2 (reduce with
 * cbct_reduce_partials).  All m entries of proj are written. */
int cbct_project(const cbct_plan* plan, const float* vol, float* proj, double* norm2_partials,
                 void* stream);

/* vol = A^T proj (mode 1, operator.py:328-341) or diag(A^T A) (mode 2,
 * operator.py:353-362; proj is ignored and may be NULL).  Every entry of vol,
 * guards included, is written (guards with 0).  scratch_proj: device workspace of
 * info.bp_scratch_floats fp32 (per-column prefix sums of the ray-length-weighted proj).  If norm2_partials != NULL it
 * receives info.bp_blocks fp64 partials of vol^2.  If col_scale != NULL the
 * result is multiplied by col_scale (Jacobi chain applyT, solvers.py:178-181). */
int cbct_backproject(const cbct_plan* plan, const float* proj, float* vol, int mode, float* scratch_proj,
                     const float* col_scale, double* norm2_partials, void* stream);

/* Sharded variants for the multi-GPU path.
 * A restricted to views [view0, view1): proj receives the (view1-view0)*nu*nv values of that view
 * block; norm2_partials (nullable) receives (view1-view0)*nu fp64 partials. */
int cbct_project_views(const cbct_plan* plan, const float* vol, float* proj, int64_t view0, int64_t view1,
                       double* norm2_partials, void* stream);
/* A^T restricted to cell rows iy in [row0, row1): vol receives (row1-row0)*nx*zstride values (that
 * slab of the device layout); col_scale is indexed like vol; norm2_partials receives
 * ceil(nx/16)*ceil((row1-row0)/16)*256 fp64 partials.  proj is the full projection set. */
int cbct_backproject_rows(const cbct_plan* plan, const float* proj, float* vol, int64_t row0, int64_t row1,
                          int mode, float* scratch_proj, const float* col_scale, double* norm2_partials,
                          void* stream);

/* ---- layout conversion (reference layout <-> internal layout) ------------ */
/* src: fp64 or fp32 (src_is_f64) reference-layout volume (nz,ny,nx) -> internal. */
int cbct_volume_to_internal(const cbct_plan* plan, const void* src, int src_is_f64, float* dst, void* stream);
/* internal -> fp64 or fp32 (dst_is_f64) reference layout (nz,ny,nx). */
int cbct_volume_from_internal(const cbct_plan* plan, const float* src, void* dst, int dst_is_f64, void* stream);
int cbct_proj_to_internal(const cbct_plan* plan, const void* src, int src_is_f64, float* dst, void* stream);
int cbct_proj_from_internal(const cbct_plan* plan, const float* src, void* dst, int dst_is_f64, void* stream);

/* ---- fused solver vector kernels (deterministic fp64 partials) ----------- */
/* Vector kernels work on flat fp32 device vectors of length n (a padded
 * internal volume or an internal projection set).  Kernels that reduce write
 * cbct_vec_blocks(n) fp64 partials (fixed element->thread map); sum them with
 * cbct_reduce_partials.  Scalars are fp64 host values, as in solvers.py. */
int cbct_vec_blocks(int64_t n);
/* CGLS volume update (solvers.py:345-346, 352; x-update deferred one iteration
 * so both fuse into one 20 B/voxel pass):  if do_x: x += alpha_prev*d ;  d = r + beta*d */
int cbct_cgls_volume_update(int64_t n, float* x, float* d, const float* r, double alpha_prev, int do_x,
                            double beta, void* stream);
/* CGLS projection update (solvers.py:353-355): e -= alpha*p, partials of e^2 (12 B/ray). */
int cbct_cgls_proj_update(int64_t n, float* e, const float* p, double alpha, double* partials, void* stream);
/* y = a*x + b*y (x NULL: y = b*y); partials of y^2 if partials != NULL. */
int cbct_axpby(int64_t n, double a, const float* x, double b, float* y, double* partials, void* stream);
/* out = a - b; partials of out^2 if partials != NULL. */
int cbct_sub(int64_t n, const float* a, const float* b, float* out, double* partials, void* stream);
/* partials of x . y */
int cbct_dot(int64_t n, const float* x, const float* y, double* partials, void* stream);
/* Device-resident CGLS loop (no host round trip per iteration; CUDA-graph capturable).
 * `scalars` is a device fp64 array: [0] ||r||^2 of the previous iteration, [1] ||r||^2
 * (written by cbct_reduce_partials after A^T), [2] ||p||^2 (after A), [3] alpha (the
 * deferred x step), [4] beta, [5] ||e||^2 (after the e update), [6] state (0 running,
 * 1 breakdown, 2 converged to [9]), [7] iterations done, [8] ||b||, [9] relative
 * discrepancy tolerance, [10] x-update flag, [16 + i] ||e||^2 of iteration i.
 * cbct_cgls_scalars evaluates the host loop's recurrences (solvers.py:339-357) in the
 * same fp64 operations -- stage 1 after A^T (beta), 2 after A (alpha), 3 after the e
 * update (history, tolerance) -- so the iterates are bitwise those of the host loop.
 * The two updates read their scalars from the array and are no-ops once state != 0. */
int cbct_cgls_scalars(double* scalars, int stage, void* stream);
int cbct_cgls_volume_update_dev(int64_t n, float* x, float* d, const float* r, const double* scalars,
                                void* stream);
int cbct_cgls_proj_update_dev(int64_t n, float* e, const float* p, const double* scalars, double* partials,
                              void* stream);
/* Device-resident LSQR (solvers.py:361-459): one A, one A^T and two fused vector passes per
 * iteration.  u and v are kept unnormalised (u = uh / nu, v = vh / nv); the U pass forms
 * uh <- tmp_m / nv - (alpha / nu) uh with tmp_m = A (scale vh), the V pass first applies the
 * previous iteration's deferred Givens update (x += a_x w ; w = vh / nv + a_w w) and then forms
 * vh <- tmp_n / nu - (beta / nv) vh with tmp_n = scale A^T uh, writing sv = scale vh for the next
 * A when scale != NULL.  Both write fp64 partials of the new vector's squared norm.
 * cbct_lsqr_scalars: stage 1 after the U pass (beta), stage 2 after the V pass (alpha, the Givens
 * rotation, the history record phibar at index 24 + iteration, breakdown / tolerance / budget
 * stops).  cbct_lsqr_flush applies the pending update once the loop has stopped.  Scalar layout:
 * 0 alpha, 1 beta, 2 rhobar, 3 phibar, 4 nu, 5 nv, 6 a_x, 7 a_w, 8 pending, 9 ||uh||^2,
 * 10 ||vh||^2, 11 state, 12 iteration, 13 ||b||, 14 tolerance, 15 max updates, 16 final a_x. */
int cbct_lsqr_u_update(int64_t n, float* uh, const float* tmp_m, const double* scalars, double* partials,
                       void* stream);
int cbct_lsqr_v_update(int64_t n, float* x, float* w, float* vh, const float* tmp_n, float* sv, const float* scale,
                       const double* scalars, double* partials, void* stream);
int cbct_lsqr_scalars(double* scalars, int stage, void* stream);
int cbct_lsqr_flush(int64_t n, float* x, const float* w, const float* vh, const double* scalars, void* stream);
/* Device-resident SIRT / PSIRT (solvers.py:505-569).  Volume pass: x += step upd (or step_vec * upd,
 * SIRT), then clip to [lo, hi] on the voxels if clip.  Projection pass: r = b - p, w = r * inv_row,
 * fp64 partials of r^2.  cbct_psirt_scalars: history record sqrt(||r||^2) / ||b|| at index
 * 8 + iteration, tolerance and budget stops.  Scalar layout: 0 ||r||^2, 1 state, 2 iteration,
 * 3 ||b||, 4 tolerance, 5 max iterations. */
int cbct_psirt_volume_update(const cbct_plan* plan, float* x, const float* upd, const float* step_vec, float step,
                             int clip, float lo, float hi, const double* scalars, void* stream);
int cbct_psirt_proj_update(int64_t m, float* r, float* w, const float* b, const float* p, const float* inv_row,
                           const double* scalars, double* partials, void* stream);
int cbct_psirt_scalars(double* scalars, void* stream);
/* Multi-GPU: *out = vals[0] + vals[1] + ... in index order (the per-rank norm partials after an
 * all_gather), the same fp64 additions as the host's rank-ordered sum. */
int cbct_sum_ranks(const double* vals, int n, double* out, void* stream);
/* Multi-GPU fused update + all-gather over NVLink peer memory: the device-scalar updates of
 * d (resp. e) that also store the rank's new slab into every rank's full-size buffer
 * (`peers`: a DEVICE array of npeers pointers from a symmetric-memory rendezvous, self
 * included) at element `offset`; d_own / e_own is the rank's slab of its own buffer.  A device
 * barrier between ranks must follow before the full vector is read. */
int cbct_cgls_volume_update_p2p(int64_t n, float* x, const float* d_own, const float* r, const double* scalars,
                                float* const* peers, int npeers, int64_t offset, void* stream);
int cbct_cgls_proj_update_p2p(int64_t n, const float* e_own, const float* p, const double* scalars,
                              double* partials, float* const* peers, int npeers, int64_t offset, void* stream);
/* Deterministic fixed-order sum of n fp64 partials into *dev_out; if host_out is
 * not NULL the result is also copied there (synchronising the stream). */
int cbct_reduce_partials(const double* partials, int32_t n, double* dev_out, double* host_out, void* stream);

/* Elementwise helpers on fp32 device vectors. */
int cbct_mul(int64_t n, const float* a, const float* b, float* out, void* stream);       /* out = a*b */
int cbct_clip(const cbct_plan* plan, float* vol, float lo, float hi, void* stream);     /* interior only */
int cbct_fill(int64_t n, float* x, float value, void* stream);
/* Fill a volume's interior with value and its guard slices with 0. */
int cbct_fill_volume(const cbct_plan* plan, float* vol, float value, void* stream);

/* ---- fp64 reference-precision path (f64.cu) ------------------------------ */
/* The same operators and vector kernels in fp64 on fp64 device buffers in the same internal
 * layouts (volume [ny][nx][zs], projections [V][nu][nv]), computed in the reference's
 * arithmetic (no FMA contraction).  CGLS / LSQR lose orthogonality after ~15-20 iterations
 * and from then on amplify any rounding difference, so only an fp64 pipeline can follow the
 * reference's fp64 iterates to 1e-3 over 40 iterations.
 * cbct_plan_enable_f64 allocates the path's one table (|r| per ray, n_rays fp64) once;
 * call it before cbct_backproject_f64.
 * cbct_project_f64: one thread per ray running the reference walk (operator.py:53-187);
 *   norm2_partials (nullable) receives cbct_f64_proj_blocks(plan) fp64 partials of proj^2.
 * cbct_backproject_f64: mode 1 A^T proj, mode 2 diag(A^T A) (proj ignored), deterministic
 *   voxel-driven gather; guards written with 0; col_scale (nullable) multiplies the result;
 *   norm2_partials receives info.bp_blocks partials. */
int cbct_plan_enable_f64(cbct_plan* plan, void* stream);
int cbct_f64_proj_blocks(const cbct_plan* plan);
int cbct_project_f64(const cbct_plan* plan, const double* vol, double* proj, double* norm2_partials,
                     void* stream);
int cbct_backproject_f64(const cbct_plan* plan, const double* proj, double* vol, int mode, const double* col_scale,
                         double* norm2_partials, void* stream);
int cbct_volume_to_internal_f64(const cbct_plan* plan, const double* src, double* dst, void* stream);
int cbct_volume_from_internal_f64(const cbct_plan* plan, const double* src, double* dst, void* stream);
int cbct_proj_to_internal_f64(const cbct_plan* plan, const double* src, double* dst, void* stream);
int cbct_proj_from_internal_f64(const cbct_plan* plan, const double* src, double* dst, void* stream);
/* fp64 vector kernels, as their fp32 counterparts above (partials: cbct_f64_vec_blocks(n)). */
int cbct_f64_vec_blocks(int64_t n);
int cbct_axpby_f64(int64_t n, double a, const double* x, double b, double* y, double* partials, void* stream);
int cbct_scale_div_f64(int64_t n, double* y, double d, double* partials, void* stream); /* y /= d */
int cbct_sub_f64(int64_t n, const double* a, const double* b, double* out, double* partials, void* stream);
int cbct_dot_f64(int64_t n, const double* x, const double* y, double* partials, void* stream);
int cbct_mul_f64(int64_t n, const double* a, const double* b, double* out, void* stream);
/* if do_x: x = x + alpha_prev*d ;  d = d*beta + r  (CGLS, solvers.py:340-341, 354-355; also LSQR's
 * x += (phi/rho) w ; w *= -(theta/rho) ; w += v, solvers.py:451-453) */
int cbct_cgls_volume_update_f64(int64_t n, double* x, double* d, const double* r, double alpha_prev, int do_x,
                                double beta, void* stream);
int cbct_fill_volume_f64(const cbct_plan* plan, double* vol, double value, void* stream);
int cbct_clip_f64(const cbct_plan* plan, double* vol, double lo, double hi, void* stream);

/* ---- phantom voxelizer ------------------------------- */
/* Replaces generate_phantom (phantom.py:87-106): sum of the intensities of the
 * ellipsoids containing each voxel centre (phantom.py:78-84), bit-identical to the
 * host generator.  `ellipsoids` is a DEVICE array of n_ell x 16 doubles per
 * ellipsoid: cx cy cz, semi-axes a b c, the row-major 3x3 rotation of
 * Ellipsoid.rotation() (phantom.py:37-40), intensity.
 * cbct_phantom writes the plan's device volume layout (guards zeroed);
 * cbct_phantom_ref writes the reference layout (nz, ny, nx), x fastest, fp32. */
int cbct_phantom(const cbct_plan* plan, const double* ellipsoids, int n_ell, float* vol, void* stream);
int cbct_phantom_ref(int64_t nx, int64_t ny, int64_t nz, const double* ellipsoids, int n_ell, float* out,
                     void* stream);
/* Same sums without the final rounding: fp64, bit-identical to the host generator for any table. */
int cbct_phantom_ref_f64(int64_t nx, int64_t ny, int64_t nz, const double* ellipsoids, int n_ell, double* out,
                         void* stream);

/* ---- reference-signature entry points (host fp64, reference layouts) ------ */
/* Drop-in for _project_kernel (operator.py:190-206). */
int cbct_ref_project(const double* vol, double* out, const double* srcs, const double* det00,
                     const double* ustep, const double* vstep, int64_t n_views, int64_t nu, int64_t nv,
                     double lo0, double lo1, double lo2, double p0, double p1, double p2, int64_t n0,
                     int64_t n1, int64_t n2);
/* Drop-in for _backproject_kernel (operator.py:209-233): out += A^T proj (mode 1)
 * or diag(A^T A) (mode 2).  n_workers is accepted for signature parity; the CUDA
 * gather is deterministic for any value. */
int cbct_ref_backproject(const double* proj, double* out, const double* srcs, const double* det00,
                         const double* ustep, const double* vstep, int64_t n_views, int64_t nu, int64_t nv,
                         double lo0, double lo1, double lo2, double p0, double p1, double p2, int64_t n0,
                         int64_t n1, int64_t n2, int64_t n_workers, int mode);

/* ---- diagnostics ---------------------------------------------------------- */
const char* cbct_last_error(void);
int cbct_version(void);
/* Number of kernel launches issued by this library since load (for the bench's gpu_launches). */
int64_t cbct_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* CBCT_H */
