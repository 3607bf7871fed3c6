"""Host-side pins of the pull SpMV layout constants (no GPU): the consumer lane
permutation in csrc/pcg.cu is a permutation of the 27 compute units and reaches the
optimum of the quarter-warp bank model of tools/pull_lane_perm.py for the 2x2
sub-block records (34/7 = 4.86 wavefronts per 16-byte instruction, found by annealing
over slot and lane permutations in tools/pull_perm_anneal.c; the identity needs 6.5),
the record offsets are a permutation of 0..35, and the 38-double record keeps block
starts 16-byte aligned."""
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


def test_table_is_optimal_in_the_bank_model():
    p = plp.table_from_source()
    assert plp.wavefronts(p) <= 34 / 7 + 1e-12
    assert plp.wavefronts(list(range(27)) + [None] * 5) > 6.0
    assert plp.split_blocks(p) <= 1


def test_record_alignment():
    src = (ROOT / "paper_2407_20026_b200" / "csrc" / "sso_internal.h").read_text()
    assert "constexpr int PULL_BLOCK = 38;" in src
    assert (38 * 8) % 16 == 0 and ((38 * 8) // 16) % 2 == 1  # 16-byte aligned, odd word stride
    assert (160 * 8) % 128 == 0  # pulled slot per node: 128-byte aligned gather4 destinations


def test_record_offsets_are_a_permutation():
    """rec_off(a, b) (csrc/sso_internal.h) restated: 2x2 sub-block (a/2, b/2) in slot
    PULL_SUB_POS[3 (b/2) + a/2], column-major inside; a bijection onto 0..35 in which each
    16-byte half holds (K[2A][c], K[2A+1][c]) -- the pair the consumers load."""
    import re
    src = (ROOT / "paper_2407_20026_b200" / "csrc" / "sso_internal.h").read_text()
    pos = int(re.search(r"PULL_SUB_POS = (0x[0-9a-f]+)ull", src).group(1), 16)
    slot = [(pos >> (4 * s)) & 15 for s in range(9)]
    assert sorted(slot) == list(range(9))
    off = {(a, b): 4 * slot[3 * (b // 2) + a // 2] + 2 * (b % 2) + (a % 2) for a in range(6) for b in range(6)}
    assert sorted(off.values()) == list(range(36))
    for (a, b), o in off.items():
        if a % 2 == 0:
            assert off[(a + 1, b)] == o + 1 and o % 2 == 0
