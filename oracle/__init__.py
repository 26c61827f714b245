"""ORACLE -- plain, slow, obviously-correct CPU implementation of the method of
arXiv 2511.16808 (shifted-Laplacian multigrid with additive Vanka smoothing and
level-dependent intergrid, as an FGMRES preconditioner for the acoustic
Helmholtz equation).

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
It shares no code with the CUDA path (``paper_2511_16808_b200/csrc``): the only
common module is the seeded input generator ``paper_2511_16808_b200.media``,
which holds none of the method's arithmetic.

Everything is complex128 / float64, assembled as SciPy sparse matrices exactly
as the paper defines the operators; each function cites the passage it
follows ("P:n" = /root/reference/PAPER.md line n).  Readings of ambiguous
passages are SURVEY.md §8(c) A1..A19, restated in DESIGN.md "Readings".

Parity status: every function here is pinned by a
``-m "not gpu"`` test in tests/test_oracle_pins.py except the ones whose header
says "parity unpinned".
"""
from .operators import (fine_operator, sigma_fields, stencil_matrix, L_stencil, M_stencil,
                        apply_helmholtz)
from .intergrid import restriction_1d, restriction, prolongation, level_scheme
from .vanka import patches, patch_counts, vanka_operator
from .hierarchy import Options, Hierarchy, build_hierarchy
from .cycle import vcycle, cycle, smooth
from .fgmres import fgmres_solve, convergence_factor
from . import lfa

__all__ = [
    "fine_operator", "sigma_fields", "stencil_matrix", "L_stencil", "M_stencil",
    "apply_helmholtz", "restriction_1d", "restriction", "prolongation", "level_scheme",
    "patches", "patch_counts", "vanka_operator", "Options", "Hierarchy", "build_hierarchy",
    "vcycle", "cycle", "smooth", "fgmres_solve", "convergence_factor", "lfa",
]
