"""Per-level damping search (scripts/damping_search.py; §5.2) on the GPU: for the
RB patch on the Table 5.2 setting, the coarse-level parameters of Table 5.1 lie in
the flat optimum of the exhaustive sweep (within one GMRES iteration of the best value), level by
level with the finer levels fixed, as the paper's procedure prescribes."""
import json
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def test_damping_search_rb_levels_1_2():
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    import damping_search as ds
    paper = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_tables.json")))["table_5_1_full"]["2d"]["rb"]
    found, sweeps, p, alpha = ds.search("rb", 128, step=0.05, lo=0.1, hi=1.0, levels=(1, 2))
    for l in (1, 2):
        best = min(its for _, its, _ in sweeps[l])
        at_paper = ds.solve(p, "rb", found[:l] + [paper[l]], l + 2, alpha)[0]
        assert at_paper <= best + 1, (l, at_paper, best)
