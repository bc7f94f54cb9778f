"""sklearn reconstructors on the GPU operator (the reference's tests/test_estimators.py):
fit/transform, equality with a direct solver call, and clone/pickle rebuilding the plan."""

import pickle

import numpy as np
import pytest
from sklearn.base import clone

from _helpers import geom_from_golden, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import paper_2110_13526_b200 as P

    d = load_golden("small_instance")
    vg, tr = geom_from_golden(d)
    op = P.CbctOperator(vg, tr)
    x = P.Volume(vg, np.random.default_rng(11).random(op.n))
    return P, op, op.project(x)


@pytest.mark.parametrize("name", ["CglsReconstructor", "LsqrReconstructor", "SirtReconstructor",
                                  "PsirtReconstructor"])
def test_fit_sets_attributes(setup, name):
    P, op, b = setup
    est = getattr(P, name)(operator=op, max_iterations=3)
    assert est.fit(b) is est
    assert est.volume_ is est.report_.final_x and est.report_.iterations == 3 and len(est.history_) >= 1
    assert isinstance(est.transform(b), P.Volume)


def test_fit_equals_direct_solver_and_clone_rebuilds_plan(setup):
    P, op, b = setup
    est = P.CglsReconstructor(operator=op, max_iterations=6).fit(b)
    rep = P.cgls(op, b, P.SolverConfig(method="cgls", max_iterations=6))
    np.testing.assert_array_equal(est.volume_.data, rep.final_x.data)
    twin = clone(est)
    assert type(twin.operator) is type(op) and twin.operator._plan.value != op._plan.value
    np.testing.assert_array_equal(twin.fit(b).volume_.data, est.volume_.data)
    op2 = pickle.loads(pickle.dumps(op))  # geometry travels; the plan is rebuilt
    np.testing.assert_array_equal(op2.project(P.Volume(op.vol_geom, np.ones(op.n))).data,
                                  op.project(P.Volume(op.vol_geom, np.ones(op.n))).data)
