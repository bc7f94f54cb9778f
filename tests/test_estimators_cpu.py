"""sklearn reconstructors (estimators.py, the reference's tests/test_estimators.py): the
parameter protocol and error contract, which need no GPU."""

import pytest
from sklearn.base import clone
from sklearn.exceptions import NotFittedError


def _classes():
    from paper_2110_13526_b200.estimators import (CglsReconstructor, LsqrReconstructor, PsirtReconstructor,
                                                  SirtReconstructor)

    return [CglsReconstructor, LsqrReconstructor, SirtReconstructor, PsirtReconstructor]


@pytest.mark.parametrize("k", range(4))
def test_params_round_trip_and_clone(k):
    cls = _classes()[k]
    est = cls(max_iterations=9, rel_discrepancy_tol=0.1)
    assert est.get_params()["max_iterations"] == 9 and est.get_params()["operator"] is None
    est.set_params(max_iterations=3)
    assert est.max_iterations == 3
    assert clone(est).get_params() == est.get_params()
    with pytest.raises(NotFittedError):
        est.history_
    with pytest.raises(ValueError):
        est.fit(None)


def test_family_specific_parameters():
    C, L, S, P = _classes()
    assert {"tikhonov_lambda", "jacobi_precondition", "jacobi_floor"} <= set(L().get_params())
    assert {"relaxation", "box_bounds"} <= set(S(box_bounds=(0.0, 1.0)).get_params())
    assert P(relaxation=1.5)._config().relaxation == 1.5 and C(jacobi_precondition=True)._config().jacobi_precondition
