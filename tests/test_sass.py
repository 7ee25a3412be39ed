"""The built library's machine code carries the Blackwell instructions the design claims (no GPU needed).

cuobjdump -sass of libshadowkv.so: every tcgen05 kernel issues UTCHMMA (tcgen05.mma), reads its TMEM
accumulator with LDTM (tcgen05.ld) and stages operands by TMA (UTMALDG); the attention kernel pulls the
value chunks with cp.async.bulk (UBLKCP) and runs QK/PV on mma.sync tiles at G >= 8 query rows;
the hot scorer keeps no local-memory spills.  DESIGN §6.
"""
import os
import shutil
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

from sass_counts import LIB, kernels, sass_counts  # noqa: E402

pytestmark = pytest.mark.skipif(shutil.which("cuobjdump") is None or not os.path.exists(LIB),
                                reason="needs cuobjdump and the built library")


@pytest.fixture(scope="module")
def counts():
    return sass_counts()


@pytest.mark.parametrize("stem", ["k_score_tc", "k_sparse_attn", "k_build_chunks", "k_gram_tc", "k_project_tc"])
def test_tcgen05_kernels_issue_umma_tmem_loads_and_tma(counts, stem):
    ks = kernels(counts, stem)
    assert ks, f"{stem} not in the library"
    for name, c in ks.items():
        assert c["UTCHMMA"] > 0, (name, c)
        assert c["LDTM"] > 0, (name, c)
        assert c["UTCBAR"] > 0, (name, c)
        assert c["UTMALDG"] > 0, (name, c)


def test_sparse_attention_gathers_by_bulk_copy_and_uses_mma_at_wide_groups(counts):
    ks = kernels(counts, "k_sparse_attn")
    assert len(ks) == 5                                   # G = 1, 2, 4, 8, 16
    for name, c in ks.items():
        assert c["UBLKCP"] > 0, (name, c)
        wide = "ILi8E" in name or "ILi16E" in name
        assert (c["HMMA"] > 0) == wide, (name, c)


def test_scorer_has_no_local_memory_traffic(counts):
    for name, c in kernels(counts, "k_score_tc").items():
        assert c["STL"] == 0 and c["LDL"] == 0, (name, c)
