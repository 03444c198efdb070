"""GPU checks of the 2D-distributed code path (paper_2601_10557_b200/dist.py) with the
CUDA ops: world size 1 in-process here; N = 2 / 4 through tools/dist_check.py under torchrun."""
import json

import numpy as np
import pytest

from conftest import GOLDEN, golden, golden_ham

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("key", ["m48_s12", "m64_s21", "m24_s100", "m32_s14", "m32_s6"])
def test_dist_path_single_gpu_matches_reference(key):
    from paper_2601_10557_b200 import SolverConfig
    from paper_2601_10557_b200.dist import solve_distributed

    kw = json.loads((GOLDEN / "meta.json").read_text())["cases"][key]
    m, seed = (int(t[1:]) for t in key.split("_"))
    a, b = golden_ham(m, seed)
    res = solve_distributed((a, b), SolverConfig(**kw), device=torch.device("cuda", 0))
    g = golden(f"solve_{key}.npz")
    assert res.converged == bool(g["converged"])
    assert abs(res.iterations_used - int(g["iterations_used"])) <= 1
    assert res.backup_events == int(g["backup_events"])
    if res.iterations_used == int(g["iterations_used"]):
        assert [t.variant for t in res.trace] == [str(x) for x in g["trace_variant"]]
    rel = np.abs(res.lambdas - g["lambdas"]) / np.abs(g["lambdas"])
    assert rel.max() <= 1e-10
    v = res.v.T.contiguous().cpu().numpy().T
    ov = np.abs(np.einsum("ij,ij->j", g["v"].conj(), v))
    assert np.abs(ov - 1).max() <= 1e-8
