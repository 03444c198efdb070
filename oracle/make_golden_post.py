"""Golden fixtures for the post-processing and CLI-bench rows (build container only; TEST
INFRASTRUCTURE): the REFERENCE's complete_spectrum / mirror_largest (solver.py:253-299) on its own
m32_s4 solve, and its `bsesolve bench` output on tests/golden/m8_s11.pchb (cli.py:291-361).

    python oracle/make_golden_post.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main() -> None:
    sys.path.insert(0, str(REF))
    import bsesolve as bs
    from bsesolve.cli import cli
    from click.testing import CliRunner

    z = np.load(OUT / "ham_m32_s4.npz")
    r = bs.solve(bs.BseHamiltonian(z["a"], z["b"]), bs.SolverConfig(nev=4, seed=9))
    cs = bs.complete_spectrum(r)
    ml = bs.mirror_largest(r)
    np.savez(OUT / "post_m32_s4.npz", lambdas=r.lambdas, v=r.v, cs_values=cs.values, cs_right=cs.right,
             cs_left=cs.left, ml_lambdas=ml.lambdas, ml_v=ml.v, ml_res=ml.residual_norms)
    tmp = Path("/tmp/bsesolve_bench_golden")
    tmp.mkdir(exist_ok=True)
    res = CliRunner().invoke(cli, ["bench", "--pchb", str(OUT / "m8_s11.pchb"), "--nev", "2", "--tol", "1e-10",
                                   "--reps", "2", "--out", str(tmp)])
    assert res.exit_code == 0, res.output
    (OUT / "m8_s11_bench.csv").write_text((tmp / "bench.csv").read_text())
    print("written", OUT / "post_m32_s4.npz", OUT / "m8_s11_bench.csv")


if __name__ == "__main__":
    main()
