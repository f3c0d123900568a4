"""Host-side plan of the Schwarz sweep's bottom levels (host/pack.cpp finish_bottom_levels):
every bottom supernode lands in exactly one level chunk per direction, a chunk's dependency
always precedes it in the ticket order (the persistent sweep's deadlock-freedom argument), and the
records fit the sweep CTA's shared block. CPU only: the symbolic plan needs no GPU."""
import os

import pytest

from paper_2512_19536_b200.simulation import Problem, SimulationConfig

CFG = dict(cells=4096, lloyd=3, degree=3, subdomains=4, coarse=-1, fiber_random=True, dt=0.01, T=0.01, tol=1e-8)

CASES = {
    "fundamental": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96"},
    "relaxed": {"PDG_ORDER": "md", "PDG_MD_RELAX": "8", "PDG_BOTTOM_KB": "160", "PDG_BOTTOM_LEVELS": "4"},
    "nested_dissection": {"PDG_ORDER": "nd", "PDG_BOTTOM_KB": "64"},
    "small_chunks": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_CHUNK_KB": "8",
                     "PDG_CHUNK_X": "256"},
    # supernodes taller than the chunk's input block stay individually scheduled (no setup error)
    "tiny_input_block": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_CHUNK_X": "64"},
    "grouped": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_BOTTOM_GROUP_MB": "1",
                "PDG_BOTTOM_GROUP_LEVELS": "2", "PDG_BOTTOM_INTERLEAVE": "2"},
    "grouped_skewed": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_BOTTOM_GROUP_MB": "1",
                       "PDG_BOTTOM_GROUP_LEVELS": "99", "PDG_BOTTOM_INTERLEAVE": "0"},
    "global_levels": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_BOTTOM_GROUP_LEVELS": "0"},
    "grouped_all_levels": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_BOTTOM_GROUP_MB": "2",
                           "PDG_BOTTOM_GROUP_LEVELS": "99", "PDG_BOTTOM_INTERLEAVE": "1"},
}


def plan(env):
    saved = {k: os.environ.get(k) for k in list(os.environ) if k.startswith("PDG_")}
    for k in saved:
        del os.environ[k]
    os.environ.update(env)
    try:
        return Problem(SimulationConfig(**CFG)).sweep_stats()
    finally:
        for k in env:
            os.environ.pop(k, None)
        os.environ.update({k: v for k, v in saved.items() if v is not None})


@pytest.mark.parametrize("name", sorted(CASES))
def test_bottom_level_plan(name):
    st = plan(CASES[name])
    assert st["plan_ok"] == 1, st
    assert 0 < st["bottom_supernodes"] <= st["supernodes"], st
    assert st["fwd_chunk_supernodes"] == st["bottom_supernodes"] == st["bwd_chunk_supernodes"], st
    assert 1 <= st["bottom_levels"] <= int(CASES[name].get("PDG_BOTTOM_LEVELS", 8)), st
    assert st["fwd_chunks"] >= st["bottom_levels"] and st["bwd_chunks"] >= 1, st


def test_bottom_levels_off_for_small_problems():
    st = plan({})
    assert st["bottom_supernodes"] == 0 and st["fwd_chunks"] == 0 and st["plan_ok"] == 1, st
