"""On-disk formats (FORMATS.md) against files written by the reference's own writers."""
import json

import numpy as np

from conftest import GOLDEN, golden, golden_ham


def test_pchb_roundtrip_and_reference_bytes(tmp_path):
    from paper_2601_10557_b200 import BseHamiltonian, fileio

    ham = fileio.read_pchb(GOLDEN / "m8_s11.pchb")
    a, b = golden_ham(8, 11)
    np.testing.assert_array_equal(ham.a, a)
    np.testing.assert_array_equal(ham.b, b)
    fileio.write_pchb(tmp_path / "x.pchb", BseHamiltonian(a, b))
    assert (tmp_path / "x.pchb").read_bytes() == (GOLDEN / "m8_s11.pchb").read_bytes()
    meta = json.loads((GOLDEN / "meta.json").read_text())
    assert fileio.digest64(tmp_path / "x.pchb") == meta["m8_s11_pchb_digest"]


def test_matrix_market_reference_bytes(tmp_path):
    from paper_2601_10557_b200 import fileio

    a, _ = golden_ham(8, 11)
    fileio.write_matrix_market(tmp_path / "A.mtx", a, comment=" resonant block, seed=11")
    assert (tmp_path / "A.mtx").read_bytes() == (GOLDEN / "m8_s11_A.mtx").read_bytes()
    np.testing.assert_array_equal(fileio.read_matrix_market(tmp_path / "A.mtx"), a)


def test_csv_and_pchv_writers_match_reference(tmp_path):
    from types import SimpleNamespace

    from paper_2601_10557_b200 import TraceRecord, fileio

    g = golden("m32_s4_result.npz")
    fileio.write_eigenvalues_csv(tmp_path / "e.csv", g["lambdas"], g["res"], "0123456789abcdef",
                                 converged=bool(g["converged"]))
    assert (tmp_path / "e.csv").read_bytes() == (GOLDEN / "m32_s4_eigenvalues.csv").read_bytes()
    trace = [TraceRecord(int(g["trace_it"][i]), int(g["trace_locked"][i]), int(g["trace_k"][i]),
                         float(g["trace_max_res"][i]), float(g["trace_min_res_unlocked"][i]),
                         float(g["trace_mu_nevex"][i]), str(g["trace_variant"][i]),
                         float(g["trace_lambda_min_m"][i]), float(g["trace_flops"][i]))
             for i in range(len(g["trace_it"]))]
    res = SimpleNamespace(trace=trace, converged=bool(g["converged"]),
                          bounds=SimpleNamespace(mu_1=float(g["mu_1"]), mu_n=float(g["mu_n"])))
    fileio.write_trace_csv(tmp_path / "t.csv", res, "0123456789abcdef")
    assert (tmp_path / "t.csv").read_bytes() == (GOLDEN / "m32_s4_trace.csv").read_bytes()
    v = fileio.read_pchv(GOLDEN / "m32_s4_v.pchv")
    fileio.write_pchv(tmp_path / "v.pchv", v)
    assert (tmp_path / "v.pchv").read_bytes() == (GOLDEN / "m32_s4_v.pchv").read_bytes()


def test_cli_parses_and_maps_validation_exit_code(tmp_path):
    from paper_2601_10557_b200.cli import main

    assert main(["solve", "--nev", "2", "--out", str(tmp_path)]) == 2  # no input -> ValidationError -> 2
