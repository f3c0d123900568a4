"""Every PDG_* tuning knob the library still reads keeps the results: each
alternative is run through tests/knob_check.py (a small solve + 3 CN steps
against the CPU oracle) in a fresh process with that environment. The knobs
select orderings, panel layout, unit sizes, L2 policy and launch modes; none
of them may change the answer beyond rounding."""
import os
import subprocess
import sys

import pytest

from tests.conftest import ROOT, gpu_available

CASES = {
    "order_md": {"PDG_ORDER": "md"},
    "order_nd": {"PDG_ORDER": "nd"},
    "md_fundamental": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_RELAX_Z": "0.1"},
    "nd_shape": {"PDG_ORDER": "nd", "PDG_ND_MERGE": "1", "PDG_ND_LEAF": "4"},
    "row_align_8": {"PDG_ROW_ALIGN": "8"},
    "small_units": {"PDG_UNIT_KB": "4", "PDG_LEAF_KB": "4"},
    "big_units": {"PDG_UNIT_MAX_KB": "256", "PDG_UNIT_KB": "256"},
    "no_prefetch": {"PDG_SWEEP_PREFETCH": "0"},
    "evict_last_prefetch": {"PDG_SWEEP_PREFETCH": "7"},
    "no_pdl": {"PDG_PDL": "0"},
    "spmv_thread_rows": {"PDG_SPMV_WARP": "0"},
    "spmv_warp_rows": {"PDG_SPMV_WARP": "1"},
    "host_loop": {"PDG_NO_GRAPH": "1"},
    "host_factor": {"PDG_HOST_FACTOR": "1"},
    "host_assembly": {"PDG_HOST_ASSEMBLY": "1"},
    "sweep_cta_64": {"PDG_SWEEP_THREADS": "64"},
    "one_cta_per_chunk": {"PDG_PERSIST": "0"},
    # bottom levels of the elimination trees solved in level chunks (off by default at this size)
    "bottom_levels": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96"},
    "bottom_levels_nd": {"PDG_BOTTOM_KB": "64", "PDG_BOTTOM_LEVELS": "3"},
    "bottom_levels_small_chunks": {"PDG_ORDER": "md", "PDG_MD_RELAX": "2", "PDG_BOTTOM_KB": "160",
                                   "PDG_BOTTOM_LEVELS": "12", "PDG_CHUNK_KB": "8", "PDG_CHUNK_X": "256"},
    "bottom_levels_cta_64": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96",
                             "PDG_SWEEP_THREADS": "64"},
    "bottom_levels_hybrid_relax": {"PDG_ORDER": "md", "PDG_RELAX_MIN_SUBTREE": "12", "PDG_BOTTOM_KB": "96"},
    "bottom_levels_grouped": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_BOTTOM_GROUP_MB": "1",
                              "PDG_BOTTOM_GROUP_LEVELS": "2", "PDG_BOTTOM_INTERLEAVE": "3"},
    "bottom_levels_global": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96", "PDG_BOTTOM_GROUP_LEVELS": "0"},
    "bottom_levels_skewed_groups": {"PDG_ORDER": "md", "PDG_MD_RELAX": "1", "PDG_BOTTOM_KB": "96",
                                    "PDG_BOTTOM_GROUP_MB": "1", "PDG_BOTTOM_GROUP_LEVELS": "3"},
    "bottom_levels_off": {"PDG_BOTTOM_KB": "0", "PDG_ORDER": "md"},
}


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
@pytest.mark.parametrize("name", sorted(CASES))
def test_knob_keeps_parity(name):
    env = {k: v for k, v in os.environ.items() if not k.startswith("PDG_")}
    env.update(CASES[name])
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "knob_check.py")], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
