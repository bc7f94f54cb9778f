"""Reference CGLS / LSQR iterates at several iteration counts, and the reference's own
reproducibility floor, at BASELINE configs 2 and 3/4 (subset).

Run in the build container only (imports the reference from ``baseline/_ref/pkg`` like
make_golden.py; ~1.5 h on 8 cores):

    NUMBA_NUM_THREADS=8 python tests/golden/make_golden_trajectory.py [check] [subset] [config2] [config2_lsqrj]

Why: CGLS and LSQR in floating point lose orthogonality once the first Ritz values
converge, and from then on any rounding difference grows roughly geometrically until it
saturates.  The reference itself shows it: changing only ``workers`` (which changes the
summation order of the backprojector's fixed-order merge, operator.py:213-233) moves its
own CGLS-40 iterate.  To make the GPU parity tests meaningful, this script records

* the reference iterate at K = 10, 20, 30, 40 (strided samples) and every history record,
  for ``workers = 8`` (the reference default) and ``workers = 5`` (same arithmetic, another
  summation order): the difference between the two is the reference's own floor;
* for LSQR + Jacobi (config 4's solver) the same at K = 40.

The loops below restate solvers.py:269-358 (cgls) and 361-459 (lsqr) statement by
statement on the reference's own operator and ``_build_chain`` (solvers.py:233-240), so
snapshots can be taken between iterations; ``check`` proves they are bitwise identical
to the reference's ``cgls``/``lsqr`` (config 1, and the subset file written by
make_golden_configs.py).
"""

from __future__ import annotations

import sys
import time

import numpy as np

from make_golden import HERE, _import_reference
from make_golden_configs import B_STRIDE, X_STRIDE, _geom_fields, _geometry, _problem

SNAPS = (10, 20, 30, 40)


def cgls_snapshots(op, b, K, snaps):
    """solvers.py:269-358 with x0 = 0, ERR = 0; returns history and {k: x after k loop iterations}."""
    from cbctkit.solvers import SolverConfig, _build_chain

    chain = _build_chain(op, SolverConfig(method="cgls", max_iterations=K))
    n, m = chain.n, chain.m
    x = np.zeros(n)
    d_x = np.zeros(n)
    r_x = np.zeros(n)
    e_b = np.zeros(m)
    p_b = np.zeros(m)
    b_eff = chain.rhs(b.data)
    nb0 = float(np.linalg.norm(b.data))
    hist, xs = [], {}
    chain.apply(x, out=p_b)
    np.subtract(b_eff, p_b, out=e_b)
    chain.applyT(e_b, out=r_x)
    nr2_old = float(r_x @ r_x)
    d_x[:] = r_x
    chain.apply(d_x, out=p_b)
    np2 = float(p_b @ p_b)
    alpha = nr2_old / np2
    x += alpha * d_x
    e_b -= alpha * p_b
    hist.append(float(np.linalg.norm(e_b)) / nb0)
    for i in range(1, K + 1):
        chain.applyT(e_b, out=r_x)
        nr2_now = float(r_x @ r_x)
        beta = nr2_now / nr2_old
        d_x *= beta
        d_x += r_x
        nr2_old = nr2_now
        chain.apply(d_x, out=p_b)
        np2 = float(p_b @ p_b)
        alpha = nr2_old / np2
        x += alpha * d_x
        e_b -= alpha * p_b
        hist.append(float(np.linalg.norm(e_b)) / nb0)
        if i in snaps:
            xs[i] = chain.x_of(x).copy()
    return np.array(hist), xs


def lsqr_snapshots(op, b, K, snaps, jacobi):
    """solvers.py:361-459 with x0 = 0, ERR = 0; x after record j is taken for j = k (k in snaps)."""
    from cbctkit.solvers import SolverConfig, _build_chain

    chain = _build_chain(op, SolverConfig(method="lsqr", max_iterations=K, jacobi_precondition=jacobi))
    n, m = chain.n, chain.m
    x = chain.z_of(np.zeros(op.n)).copy()
    b_eff = chain.rhs(b.data)
    nb0 = float(np.linalg.norm(b.data))
    u = np.empty(m)
    chain.apply(x, out=u)
    np.subtract(b_eff, u, out=u)
    beta = float(np.linalg.norm(u))
    u /= beta
    v = np.empty(n)
    chain.applyT(u, out=v)
    alpha = float(np.linalg.norm(v))
    v /= alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    tmp_m = np.empty(m)
    tmp_n = np.empty(n)
    hist, xs = [], {}
    for updates in range(K + 1):
        chain.apply(v, out=tmp_m)
        u *= -alpha
        u += tmp_m
        beta = float(np.linalg.norm(u))
        u /= beta
        chain.applyT(u, out=tmp_n)
        v *= -beta
        v += tmp_n
        alpha = float(np.linalg.norm(v))
        v /= alpha
        rho = np.hypot(rhobar, beta)
        c = rhobar / rho
        s = beta / rho
        theta = s * alpha
        rhobar = -c * alpha
        phi = c * phibar
        phibar = s * phibar
        x += (phi / rho) * w
        w *= -(theta / rho)
        w += v
        hist.append(phibar / nb0)
        if updates in snaps:
            xs[updates] = chain.x_of(x).copy()
    return np.array(hist), xs


def _store(out, key, hist, xs):
    out[f"{key}_hist"] = hist
    for k, x in xs.items():
        out[f"{key}_x{k}_sample"] = x[::X_STRIDE].copy()
        out[f"{key}_x{k}_norm"] = np.array(np.linalg.norm(x))


def check():
    """Bitwise equality of the restated loops with the reference's cgls / lsqr (config 1)."""
    from cbctkit.operator import CbctOperator
    from cbctkit.solvers import SolverConfig, cgls, lsqr

    vg, tr = _geometry(64, 90, 128, 96)
    _, b = _problem(vg, tr)
    op = CbctOperator(vg, tr, workers=8)
    h, xs = cgls_snapshots(op, b, 12, (12,))
    rep = cgls(op, b, SolverConfig(method="cgls", max_iterations=12))
    assert np.array_equal(xs[12], rep.final_x.data), "cgls restatement is not bitwise"
    assert np.array_equal(h, [r.rel_discrepancy for r in rep.history])
    h, xs = lsqr_snapshots(op, b, 12, (12,), True)
    rep = lsqr(op, b, SolverConfig(method="lsqr", max_iterations=12, jacobi_precondition=True))
    assert np.array_equal(xs[12], rep.final_x.data), "lsqr restatement is not bitwise"
    assert np.array_equal(h, [r.rel_discrepancy for r in rep.history])
    sub = HERE / "config34_subset.npz"
    if sub.exists():
        with np.load(sub) as z:
            vg, tr = _geometry(512, 720, 616, 480, stride=8, zslab=(240, 32))
            _, b = _problem(vg, tr)
            assert np.array_equal(b.data[::B_STRIDE], z["b_sample"])
    print("check: restated cgls / lsqr are bitwise equal to the reference")


def _trajectories(name, vg, tr, lsqr_too, cgls_too=True):
    from cbctkit.operator import CbctOperator

    _, b = _problem(vg, tr)
    out = dict(_geom_fields(vg, tr), x_stride=np.array(X_STRIDE), b_stride=np.array(B_STRIDE),
               b_sample=b.data[::B_STRIDE].copy(), b_norm=np.array(np.linalg.norm(b.data)),
               snaps=np.array(SNAPS))
    for w in (8, 5):
        op = CbctOperator(vg, tr, workers=w)
        if cgls_too:
            t = time.perf_counter()
            _store(out, f"cgls_w{w}", *cgls_snapshots(op, b, 40, SNAPS))
            print(f"  cgls w={w}: {time.perf_counter() - t:.0f} s", flush=True)
        if lsqr_too:
            t = time.perf_counter()
            _store(out, f"lsqrj_w{w}", *lsqr_snapshots(op, b, 40, SNAPS, True))
            print(f"  lsqrj w={w}: {time.perf_counter() - t:.0f} s", flush=True)
        np.savez_compressed(HERE / f"{name}_trajectory.npz", **out)


def subset():
    vg, tr = _geometry(512, 720, 616, 480, stride=8, zslab=(240, 32))
    _trajectories("config34_subset", vg, tr, True)


def config2():
    vg, tr = _geometry(256, 360, 512, 384)
    _trajectories("config2", vg, tr, False)


def config2_lsqrj():
    """LSQR + Jacobi (config 4's solver) on BASELINE config 2 in full (~1 h on 8 cores)."""
    vg, tr = _geometry(256, 360, 512, 384)
    _trajectories("config2_lsqrj", vg, tr, True, cgls_too=False)


def main(argv):
    if argv[:1] == ["compact"]:
        for name in argv[1:]:
            compact(name)
        return
    _import_reference()
    for w in argv or ["check", "subset", "config2"]:
        print(w, flush=True)
        {"check": check, "subset": subset, "config2": config2, "config2_lsqrj": config2_lsqrj}[w]()
        if w != "check":
            compact({"subset": "config34_subset"}.get(w, w))


def compact(name):
    """Shrink <name>_trajectory.npz for the repository: the workers=8 samples are kept in fp32
    (the tests compare at 1e-3), the workers=5 run is reduced to its floor -- the rel-L2 of
    its samples against the workers=8 samples, taken in fp64 before the narrowing."""
    path = HERE / f"{name}_trajectory.npz"
    with np.load(path) as z:
        d = {k: z[k] for k in z.files}
    out = {}
    for k, v in d.items():
        if "_w5_x" in k:
            if k.endswith("_sample"):
                ref = d[k.replace("_w5_", "_w8_")]
                key = k.replace("_w5_", "_").replace("_sample", "_floor")
                out[key] = np.array(np.linalg.norm(v - ref) / np.linalg.norm(ref))
            continue
        out[k] = v.astype(np.float32) if ("_w8_x" in k and k.endswith("_sample")) else v
    np.savez_compressed(path, **out)
    print(f"compacted {path.name}: {path.stat().st_size / 1024:.0f} KiB")


if __name__ == "__main__":
    main(sys.argv[1:])
