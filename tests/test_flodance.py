"""FLODANCE: the scaling-law fit over the engine's prefix log-determinants.

Pinned to the unmodified reference's outputs (tests/golden/flodance.*, made by
tests/golden/make_flodance_golden.py from oocdet.flodance on oracle prefixes of seeded
BASELINE-family matrices), plus the model identities the reference's own tests check
(tests/test_flodance.py there) restated here.  Host-only: runs in the CPU suite."""

import json
import math
import os

import numpy as np
import pytest
from scipy.special import gammaln
from scipy.stats import norm

from paper_2503_04424_b200 import (
    ConditioningError,
    FlodanceFit,
    PrefixWriter,
    build_design,
    extract_l,
    fit_design,
    fit_prefix,
    predict,
    predict_interval,
    scaling_ratio_trace,
    select_burn_in,
)
from paper_2503_04424_b200.cli import main

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def fgold():
    with open(os.path.join(HERE, "flodance.json")) as f:
        meta = json.load(f)
    return meta, np.load(os.path.join(HERE, "flodance.npz"))


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.abs(b)))) if a.size else 0.0


def test_fits_and_predictions_match_reference(fgold):
    meta, z = fgold
    assert len(meta["cases"]) >= 7
    for c in meta["cases"]:
        fit = fit_prefix(z["seq_" + c["seq"]], c["d"], c["n0"], c["ns"], c["q"])
        ref = c["fit"]
        assert (fit.n0, fit.ns, fit.q) == (ref["n0"], ref["ns"], ref["q"])
        assert fit.c0 == pytest.approx(ref["c0"], rel=1e-9, abs=1e-12), c["key"]
        np.testing.assert_allclose(fit.nu, ref["nu"], rtol=1e-9, atol=1e-12, err_msg=c["key"])
        assert fit.sigma_hat == pytest.approx(ref["sigma_hat"], rel=1e-9, abs=1e-14)
        assert fit.anchor == ref["anchor_L"]  # L_{n0} is a plain division: bit-equal
        L, e = predict(fit, np.arange(c["ns"] + 1, c["n"] + 1))
        assert _rel(L, z[c["key"] + "_L_hat"]) <= 1e-12, c["key"]
        assert _rel(e, z[c["key"] + "_ell_hat"]) <= 1e-12, c["key"]
        np.testing.assert_allclose(fit.residuals, z[c["key"] + "_residuals"], rtol=0, atol=1e-10)
        lo, hi = predict_interval(fit, c["n"], 0.9)
        assert _rel([lo, hi], c["interval90"]) <= 1e-12


def test_burn_in_and_traces_match_reference(fgold):
    meta, z = fgold
    for b in meta["burn_in"]:
        assert select_burn_in(z["seq_" + b["seq"]], b["d"], b["ns"], b["q"], candidates=(1, 10, 50, 100)) == b["n0"]
    for name in ("rbf600", "ntk500"):
        for d in (1, 2):
            np.testing.assert_array_equal(scaling_ratio_trace(z["seq_" + name], d), z[f"{name}_trace_d{d}"])


def _model_prefix(fit, upto):
    n = np.arange(1, upto + 1)
    _, ell = predict(fit, n)
    ell = np.array(ell)
    ell[fit.n0 - 1] = fit.n0 * fit.anchor  # the regression is anchored at the observed L_{n0}
    return ell


def test_exact_model_recovered_and_extrapolated():
    true = FlodanceFit(n0=2, ns=60, q=0, c0=1.5, nu=np.array([0.7]), sigma_hat=0.0, anchor=-1.0)
    got = fit_prefix(_model_prefix(true, 60), 1, 2, 60, 0)
    assert got.c0 == pytest.approx(1.5, rel=1e-8) and got.nu[0] == pytest.approx(0.7, rel=1e-8)
    assert predict(got, 600)[0] == pytest.approx(predict(true, 600)[0], abs=1e-10)
    assert got.sigma_hat < 1e-9


def test_design_entries_and_log_factorials():
    X, y = build_design(np.zeros(10), 1, 10, 2)
    assert X[0, 0] == 1.0  # n_j = 2
    assert X[0, 1] == pytest.approx(-math.log(2.0), rel=1e-12)
    assert X[0, 2] == pytest.approx(-math.log(2.0) / 2, rel=1e-12)
    assert np.all(y == 0)
    X, _ = build_design(np.zeros(20), 1, 20, 0)
    for row, nj in enumerate(range(2, 21)):
        assert X[row, 1] == pytest.approx(-math.log(math.factorial(nj)) / math.sqrt(nj - 1), rel=1e-13)


def test_extract_and_ratio_trace_definitions():
    ell = np.arange(1, 41, dtype=float) * math.log(3.0)
    np.testing.assert_allclose(extract_l(ell, 2, 1, 20), 2 * math.log(3.0))
    n = np.arange(1, 31)
    np.testing.assert_allclose(scaling_ratio_trace(np.cumsum(-np.log(n)), 1), -np.log(n[1:]), rtol=1e-12)
    with pytest.raises(ValueError):
        extract_l(np.zeros(10), 3, 1, 5)
    with pytest.raises(ValueError):
        build_design(np.zeros(4), 1, 4, 2)
    with pytest.raises(ValueError):
        scaling_ratio_trace(np.zeros(1), 1)


def test_rank_deficient_and_zero_columns_raise():
    X = np.ones((10, 3))
    X[:, 2] = 2 * X[:, 1]
    with pytest.raises(ConditioningError):
        fit_design(X, np.ones(10))
    X = np.ones((10, 2))
    X[:, 1] = 0.0
    with pytest.raises(ConditioningError, match="column 1"):
        fit_design(X, np.ones(10))


def test_interval_arithmetic():
    fit = FlodanceFit(n0=1, ns=50, q=0, c0=0.0, nu=np.zeros(1), sigma_hat=1.0, anchor=0.0)
    lo, hi = predict_interval(fit, 101, 0.95)
    assert hi - lo == pytest.approx(2 * norm.ppf(0.975) * 10.0, rel=1e-12)
    with pytest.raises(ValueError):
        predict_interval(fit, 101, 1.0)
    zero = FlodanceFit(n0=1, ns=50, q=1, c0=0.0, nu=np.zeros(2), sigma_hat=0.0, anchor=7.5)
    assert predict(zero, 123) == (7.5, 123 * 7.5)
    assert predict_interval(zero, 100)[0] == predict_interval(zero, 100)[1]


def test_cli_flodance_from_sidecar(tmp_path, capsys):
    """`flodance` on a MDPREFIX sidecar (host only: the sidecar is written directly)."""
    j = np.arange(1, 81, dtype=np.float64)
    ell = j * (1.0 - 0.3 * gammaln(j + 1) / j ** 2) + 1e-4 * np.cos(j)
    side = tmp_path / "s.pfx"
    with PrefixWriter(side) as w:
        w.append(ell, np.ones(len(ell), np.int64))
    trace = tmp_path / "t.csv"
    code = main(["flodance", "--prefix", str(side), "--d", "1", "--n0", "5", "--ns", "70", "--q", "1",
                 "--predict", "80", "--interval", "0.9", "--trace-out", str(trace), "--json"])
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert code == 0
    fit = fit_prefix(ell, 1, 5, 70, 1)
    assert out["c0"] == fit.c0 and out["logdet_hat"] == float(predict(fit, 80)[1])
    assert out["interval"]["lower"] <= out["logdet_hat"] <= out["interval"]["upper"]
    lines = trace.read_text().strip().splitlines()
    assert lines[0] == "n,log_ratio" and len(lines) == 80
