"""Host-side pins of the pull SpMV layout constants (no GPU): the consumer lane
permutation in csrc/pcg.cu is a permutation of the 27 compute units and keeps every
16-byte shared-memory access of an interior node conflict-free under the quarter-warp
bank model of tools/pull_lane_perm.py (4 wavefronts per instruction; the identity
needs 5.6), and the 38-double record keeps block starts 16-byte aligned."""
import importlib.util
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
spec = importlib.util.spec_from_file_location("pull_lane_perm", ROOT / "tools" / "pull_lane_perm.py")
plp = importlib.util.module_from_spec(spec)
spec.loader.exec_module(plp)


def test_table_is_a_unit_permutation():
    p = plp.table_from_source()
    assert len(p) == 32
    assert sorted(u for u in p if u is not None) == list(range(27))


def test_table_is_conflict_free_in_the_bank_model():
    p = plp.table_from_source()
    assert plp.wavefronts(p) == 4.0
    assert plp.wavefronts(list(range(27)) + [None] * 5) > 5.0
    assert plp.split_blocks(p) <= 1


def test_record_alignment():
    src = (ROOT / "paper_2407_20026_b200" / "csrc" / "sso_internal.h").read_text()
    assert "constexpr int PULL_BLOCK = 38;" in src
    assert (38 * 8) % 16 == 0 and ((38 * 8) // 16) % 2 == 1  # 16-byte aligned, odd word stride
    assert (160 * 8) % 128 == 0  # pulled slot per node: 128-byte aligned gather4 destinations
