"""CLI parity with the reference's memdet / cost subcommands (reference tests/test_cli.py)."""

import json

import numpy as np
import pytest

from paper_2503_04424_b200 import gen, write_matrix
from paper_2503_04424_b200.cli import main, parse_size

MEMDET_KEYS = {"schema_version", "logabsdet", "sign", "n_b", "b", "blocks_read", "blocks_written",
               "scratch_slots", "wall_seconds"}


@pytest.mark.parametrize("text,expect", [("1024", 1024), ("4K", 4096), ("2m", 2 << 20), ("1G", 1 << 30),
                                         ("1.5k", 1536), ("8kb", 8192)])
def test_parse_size(text, expect):
    assert parse_size(text) == expect


def test_cost_json(capsys):
    assert main(["cost", "--m", "4096", "--nb", "4", "--case", "sym", "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["schema_version"] == 1 and (out["blocks_read"], out["blocks_written"], out["scratch_slots"]) == (18, 8, 6)


def test_cost_defaults_to_generic_with_exact_integers(capsys):
    """`cost --m M --nb N` without --case is the generic case, and exact counts are JSON ints
    (reference cli.py:276-279, cost.py:58-60)."""
    from paper_2503_04424_b200.cost import predicted_cost

    assert main(["cost", "--m", "4096", "--nb", "4", "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    pc = predicted_cost(4096, 4, "generic")
    assert out["case"] == "generic"
    assert isinstance(out["total_flops"], int) and out["total_flops"] == pc.total_flops
    for name, op in out["operations"].items():
        assert all(isinstance(op[k], int) for k in ("count", "flops_per_op", "total")), (name, op)
        assert op["total"] == getattr(pc, name).total


def test_usage_and_io_exit_codes(tmp_path, capsys):
    p = tmp_path / "g.mdm"
    write_matrix(p, gen.random_spd(8, seed=1), "generic")
    assert main(["memdet", "--in", str(p), "--assume", "spd", "--num-blocks", "1"]) == 2  # generic file
    assert main(["memdet", "--in", str(p), "--assume", "gen", "--num-blocks", "1",
                 "--prefix-out", str(tmp_path / "x.pfx")]) == 2  # no prefixes for generic (cli.py:85-88)
    bad = tmp_path / "bad.mdm"
    bad.write_bytes(b"not a matrix file at all" * 4)
    assert main(["memdet", "--in", str(bad), "--assume", "spd", "--num-blocks", "1"]) == 4
    assert main(["memdet", "--in", str(tmp_path / "missing.mdm"), "--assume", "spd", "--num-blocks", "1"]) == 4


def test_gen_writes_memdet01(tmp_path, capsys):
    out = tmp_path / "k.mdm"
    assert main(["gen", "--kind", "rbf", "--n", "64", "--out", str(out), "--json"]) == 0
    meta = json.loads(capsys.readouterr().out)
    assert meta["m"] == 64 and meta["symmetry"] == "spd"
    raw = open(out, "rb").read()
    assert raw[:8] == b"MEMDET01" and len(raw) == 64 + 64 * 64 * 8


@pytest.mark.gpu
def test_memdet_json_on_gpu(tmp_path, capsys):
    a = gen.random_spd(300, seed=4)
    p = tmp_path / "s.mdm"
    write_matrix(p, a, "spd")
    assert main(["memdet", "--in", str(p), "--assume", "spd", "--num-blocks", "3", "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert MEMDET_KEYS <= set(out)
    assert out["logabsdet"] == pytest.approx(float(np.linalg.slogdet(a)[1]), rel=1e-10)
    assert main(["memdet", "--in", str(p), "--assume", "sym", "--num-blocks", "3", "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["sign"] == 1 and out["logabsdet"] == pytest.approx(float(np.linalg.slogdet(a)[1]), rel=1e-10)
    bad = tmp_path / "ind.mdm"
    write_matrix(bad, gen.random_symmetric(50, seed=2), "symmetric")
    assert main(["memdet", "--in", str(bad), "--assume", "spd", "--num-blocks", "2"]) == 3  # NotSpd


@pytest.mark.gpu
def test_pipeline_json_on_gpu(tmp_path, capsys):
    """`pipeline` (reference cli.py:169-199): generate, factor on the engine, fit, extrapolate."""
    from oracle import memdet_oracle as O
    from paper_2503_04424_b200 import fit_prefix, predict

    out_path = tmp_path / "k.mdm"
    assert main(["pipeline", "--kind", "rbf", "--n", "400", "--seed", "3", "--out", str(out_path),
                 "--assume", "spd", "--num-blocks", "2", "--n0", "5", "--ns", "300", "--q", "1", "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["command"] == "pipeline" and {"matrix", "memdet", "flodance", "rel_error"} <= set(out["outputs"])
    ref, _ = O.memdet_cholesky(gen.rbf(400, seed=3), 2)
    assert out["outputs"]["memdet"]["logabsdet"] == pytest.approx(float(ref[-1]), rel=1e-10)
    fit = fit_prefix(ref, 1, 5, 300, 1)
    assert out["outputs"]["flodance"]["logdet_hat"] == pytest.approx(float(predict(fit, 400)[1]), rel=1e-8)
    assert out["outputs"]["rel_error"] >= 0.0


@pytest.mark.gpu
def test_memdet_gen_json_on_gpu(tmp_path, capsys):
    """`memdet --assume gen` runs the LU path (reference cli.py:81-104)."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal((200, 200)) + 30 * np.eye(200)
    a[0] *= -1
    p = tmp_path / "g.mdm"
    write_matrix(p, a, "generic")
    assert main(["memdet", "--in", str(p), "--assume", "gen", "--num-blocks", "3", "--json"]) == 0
    out = json.loads(capsys.readouterr().out)
    sign, ld = np.linalg.slogdet(a)
    assert out["sign"] == int(sign) and out["logabsdet"] == pytest.approx(ld, rel=1e-10)
    assert (out["n_b"], out["blocks_read"], out["blocks_written"], out["scratch_slots"]) == (3, 13, 4, 4)
