"""Host setup against the oracle (no GPU): the product's assembly of M, A and
K (assembly.cpp:89-202) is bitwise the oracle's, E (schwarz.cpp:13-77) is
exact and K0 = E^T K E (schwarz.cpp:141) agrees to rounding. Pins the
parallel assembly / scatter / K0 accumulation to the serial order."""
import numpy as np
import pytest

from paper_2512_19536_b200.simulation import Problem, SimulationConfig
from tests.oracle_binding import oracle_for

CASES = [dict(cells=512, degree=2, subdomains=8, coarse=-1, fiber_random=True),
         dict(cells=300, degree=3, subdomains=6, coarse=4, q=2),
         dict(cells=256, degree=1)]


@pytest.mark.parametrize("kw", CASES, ids=lambda k: f"{k['cells']}-p{k['degree']}")
def test_assembly_bitwise_and_coarse_space(kw):
    cfg = SimulationConfig(**kw)
    P = Problem(cfg)
    orc, _ = oracle_for(cfg)
    for w in ("K", "M", "A"):
        a, b = P.export(w).tocsr(), orc.export(w).tocsr()
        a.sort_indices()
        b.sort_indices()
        assert a.shape == b.shape and np.array_equal(a.indptr, b.indptr) and np.array_equal(a.indices, b.indices)
        assert np.array_equal(a.data, b.data), w
    E, Eo = P.export("E").toarray(), orc.export("E").toarray()
    assert np.array_equal(E, Eo)
    K0, K0o = P.export("K0").toarray(), orc.export("K0").toarray()
    assert np.abs(K0 - K0o).max() <= 1e-13 * np.abs(K0o).max()
