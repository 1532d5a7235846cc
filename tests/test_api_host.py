"""Host-side API parity with the reference `sso` package (no GPU needed).

Mirrors the reference's own unit tests for the pieces that are plain host
logic: parameter validation, the scalar update rule, the benchmark registry
metadata, layouts, schedules, partitioning, records, and the argument checks
that must fire before any device work.
"""

import warnings

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2110_01470_b200 as psso
from paper_2110_01470_b200 import sharded

EXPECTED_BOUNDS = {
    "f1": (-5.12, 5.12), "f2": (-5.12, 5.12), "f3": (-65.536, 65.536), "f4": (-2.048, 2.048),
    "f5": (-5.12, 5.12), "f6": (-32.768, 32.768), "f7": (-600.0, 600.0), "f8": (-4.0, 5.0),
    "f9": (-5.12, 5.12),
}


class TestSsoParams:  # reference test_core.py:24-49
    def test_threshold_ordering_enforced(self):
        with pytest.raises(ValueError, match="thresholds"):
            psso.SsoParams(cw=0.5, cp=0.4, cg=0.8, var_min=0, var_max=1, nsol=1, nvar=1, niter=1)
        with pytest.raises(ValueError, match="thresholds"):
            psso.SsoParams(cw=0.1, cp=0.2, cg=1.2, var_min=0, var_max=1, nsol=1, nvar=1, niter=1)

    def test_degenerate_interval_rejected(self):
        with pytest.raises(ValueError, match="var_min < var_max"):
            psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=2.0, var_max=2.0, nsol=1, nvar=1, niter=1)

    @pytest.mark.parametrize("field", ["nsol", "nvar", "niter"])
    def test_counts_must_be_positive(self, field):
        kw = dict(cw=0.3, cp=0.6, cg=0.8, var_min=0, var_max=1, nsol=2, nvar=2, niter=2)
        kw[field] = 0
        with pytest.raises(ValueError, match=field):
            psso.SsoParams(**kw)

    def test_equal_thresholds_are_legal(self):
        p = psso.SsoParams(cw=1.0, cp=1.0, cg=1.0, var_min=0, var_max=1, nsol=1, nvar=1, niter=1)
        assert p.cw == p.cg == 1.0 and p.span == 1.0


class TestStepUpdate:  # reference test_core.py:52-104
    P = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-5.12, var_max=5.12, nsol=1, nvar=1, niter=1)

    def test_branches(self):
        f = psso.step_update_variable
        assert f(1.0, 2.0, 3.0, 0.10, 4.0, self.P) == 1.0
        assert f(1.0, 2.0, 3.0, 0.45, 4.0, self.P) == 2.0
        assert f(1.0, 2.0, 3.0, 0.70, 4.0, self.P) == 3.0
        assert f(1.0, 2.0, 3.0, 0.95, 4.0, self.P) == 4.0

    @pytest.mark.parametrize("u", [-0.01, 1.0, 1.5, float("nan")])
    def test_branch_deviate_domain_checked(self, u):
        with pytest.raises(ValueError, match="branch deviate"):
            psso.step_update_variable(1.0, 2.0, 3.0, u, 4.0, self.P)

    @given(u=st.floats(min_value=0.0, max_value=1.0, exclude_max=True),
           th=st.tuples(st.floats(0, 1), st.floats(0, 1), st.floats(0, 1)))
    @settings(max_examples=200, deadline=None)
    def test_integer_threshold_compare_is_exact(self, u, th):
        """The kernels compare k = h >> 11 against ceil(c * 2^53); equivalent to u < c."""
        import math

        cw, cp, cg = sorted(th)
        k = math.floor(u * 2.0**53)
        uq = k * 2.0**-53  # every reference deviate has this form
        for c in (cw, cp, cg):
            K = min(max(math.ceil(c * 2.0**53), 0), 2**53)
            assert (uq < c) == (k < K)


class TestRegistry:  # reference test_benchmarks.py
    def test_suite_at_dimension_four_has_all_nine(self):
        suite = psso.list_suite(4)
        assert [fn.id for fn in suite] == list(psso.FUNCTION_IDS)
        for fn in suite:
            assert fn.bounds == EXPECTED_BOUNDS[fn.id]

    def test_powell_dimension_rules(self):
        with pytest.raises(ValueError, match="divisible by 4"):
            psso.make_function("f8", 50, strict=True)
        with pytest.warns(UserWarning, match="first 48"):
            fn = psso.make_function("f8", 50)
        assert fn.truncated_to == 48

    def test_suite_omits_powell_at_indivisible_dimension(self):
        with pytest.warns(UserWarning, match="omitting f8"):
            suite = psso.list_suite(50)
        assert [fn.id for fn in suite] == [f for f in psso.FUNCTION_IDS if f != "f8"]
        with pytest.raises(ValueError, match="divisible by 4"):
            psso.list_suite(50, strict=True)

    def test_unknown_id_and_bad_dims(self):
        with pytest.raises(ValueError, match="unknown function id"):
            psso.make_function("f10", 8)
        with pytest.raises(ValueError, match="f4 needs dimension"):
            psso.make_function("f4", 1)
        with pytest.raises(ValueError, match="dimension must be positive"):
            psso.make_function("f1", 0)

    def test_deviation_ledger(self):
        assert set(psso.DEVIATIONS) == {"f3", "f5", "f6", "f8", "f9"}

    def test_reference_points(self):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            for fn in psso.list_suite(48):
                assert np.all(fn.reference_point >= fn.var_min)
                assert np.all(fn.reference_point <= fn.var_max)
        f9 = psso.make_function("f9", 50)
        xs = np.linspace(-5.12, 5.12, 400001)
        h = xs * np.sin(np.sqrt(np.abs(xs)))
        assert f9.reference_value == pytest.approx(418.9829 * 50 - 50 * h.max(), abs=1e-6)

    def test_dimension_mismatch_rejected_before_device(self):
        fn = psso.make_function("f1", 10)
        with pytest.raises(ValueError, match="dimension 10"):
            fn(np.zeros(9))


class TestLayoutAndSchedule:  # reference test_parallel.py:289-333
    def test_identity_conversion(self):
        m = np.arange(6.0).reshape(2, 3)
        assert psso.convert_layout(m, psso.LayoutMode.PARTICLE_MAJOR, psso.LayoutMode.PARTICLE_MAJOR) is m

    def test_interleaved_storage_order(self):
        m = np.array([[1.0, 2.0], [3.0, 4.0]])
        inter = psso.convert_layout(m, psso.LayoutMode.PARTICLE_MAJOR, psso.LayoutMode.INTERLEAVED)
        assert np.array_equal(inter, m) and inter.flags["F_CONTIGUOUS"]
        assert list(inter.ravel(order="K")) == [1.0, 3.0, 2.0, 4.0]

    def test_dimension_mismatch_rejected(self):
        with pytest.raises(ValueError, match="2-D"):
            psso.convert_layout(np.zeros(5), psso.LayoutMode.PARTICLE_MAJOR, psso.LayoutMode.INTERLEAVED)

    def test_schedule_validation(self):
        assert psso.Schedule(kind=psso.ScheduleKind.PARALLEL, workers=4).workers == 4
        with pytest.raises(ValueError, match="workers"):
            psso.Schedule(kind=psso.ScheduleKind.PARALLEL, workers=0)
        assert str(psso.ScheduleKind.PARALLEL) == "parallel"
        assert str(psso.LayoutMode.INTERLEAVED) == "interleaved"


class TestPartition:  # reference parallel.py:147-149
    @given(nsol=st.integers(1, 5000), parts=st.integers(1, 64))
    @settings(max_examples=200, deadline=None)
    def test_contiguous_disjoint_cover(self, nsol, parts):
        ranges = psso.partition(nsol, parts)
        assert ranges[0][0] == 0 and ranges[-1][1] == nsol
        for (a, b), (c, d) in zip(ranges, ranges[1:]):
            assert b == c and a < b
        edges = np.linspace(0, nsol, parts + 1).astype(int)
        ref = [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:]) if b > a]
        assert ranges == ref

    def test_rejects_zero_parts(self):
        with pytest.raises(ValueError):
            sharded.partition(10, 0)


def test_run_record_scalar_view_and_equality():
    r = psso.RunRecord(0, psso.ScheduleKind.PARALLEL, "f5", 15, 20, 40, 0.3, 0.6, 0.8, 1, 2.5,
                       0.25, best_position=np.zeros(3), trajectory=np.ones(4))
    s = psso.RunRecord(0, psso.ScheduleKind.PARALLEL, "f5", 15, 20, 40, 0.3, 0.6, 0.8, 1, 2.5, 0.25)
    assert r == s  # array extras excluded from equality
    assert list(r.scalar_row()) == ["run_id", "schedule", "function", "nsol", "nvar", "niter",
                                    "cw", "cp", "cg", "seed", "best_fitness", "wall_time_s"]


def test_run_parallel_validates_before_device():
    fn = psso.make_function("f1", 4)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=4, nvar=4, niter=2)
    with pytest.raises(ValueError, match="workers"):
        psso.run_parallel(p, fn, seed=0, workers=0)
    with pytest.raises(ValueError):
        psso.run_parallel(p, fn, seed=0, layout="diagonal")


def test_nonfinite_error_message():
    e = psso.NonFiniteFitnessError(float("inf"), 2, 7)
    assert "particle 2" in str(e) and "iteration 7" in str(e)
    assert "during initialization" in str(psso.NonFiniteFitnessError(float("nan"), 0))


def test_product_has_no_cpu_fallback(monkeypatch):
    """Without a GPU the engine refuses to run instead of computing on the host."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    fn = psso.make_function("f1", 4)
    p = psso.SsoParams(cw=0.3, cp=0.6, cg=0.8, var_min=-1, var_max=1, nsol=4, nvar=4, niter=2)
    with pytest.raises(RuntimeError, match="CUDA"):
        psso.run_parallel(p, fn, seed=0)
    with pytest.raises(RuntimeError, match="CUDA"):
        fn(np.zeros(4))
    with pytest.raises(RuntimeError, match="CUDA"):
        psso.RngStream(0).uniform(psso.SubStream.BRANCH, 0, 0, 0)
