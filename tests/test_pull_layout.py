"""Host-side pins of the pull SpMV layout constants (no GPU): the consumer lane
permutation in csrc/pcg.cu is a permutation of the 27 compute units and reaches the
best value found for the quarter-warp bank model of tools/pull_lane_perm.py with the 2x2
sub-block records (30/7 = 4.29 wavefronts per 16-byte instruction, annealing over the
sub-block slot order, the pad position and the lane table in tools/pull_perm_anneal.c;
the identity table needs 6.0), the record offsets place the 36 values on distinct
doubles outside one 16-byte pad word, and the 38-double record keeps block starts
16-byte aligned."""
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
    assert plp.wavefronts(p) <= 30 / 7 + 1e-12
    assert plp.wavefronts(list(range(27)) + [None] * 5) > 6.0
    assert plp.split_blocks(p) <= 1


def test_record_alignment():
    src = (ROOT / "paper_2407_20026_b200" / "csrc" / "sso_internal.h").read_text()
    assert "constexpr int PULL_BLOCK = 38;" in src
    assert (38 * 8) % 16 == 0 and ((38 * 8) // 16) % 2 == 1  # 16-byte aligned, odd word stride
    assert (160 * 8) % 128 == 0  # pulled slot per node: 128-byte aligned gather4 destinations


def test_record_offsets_are_a_permutation():
    """rec_off(a, b) (csrc/sso_internal.h) restated: 2x2 sub-block (a/2, b/2) in slot
    q = PULL_SUB_POS[3 (b/2) + a/2] at double 4 q (+ 2 from the pad word on), column-major
    inside: the 36 values land on distinct doubles of the 38, the other two form one aligned
    16-byte pad word, and each 16-byte half holds (K[2A][c], K[2A+1][c])."""
    import re
    src = (ROOT / "paper_2407_20026_b200" / "csrc" / "sso_internal.h").read_text()
    pos = int(re.search(r"PULL_SUB_POS = (0x[0-9a-f]+)ull", src).group(1), 16)
    gap = int(re.search(r"PULL_SUB_GAP = (\d+);", src).group(1))
    slot = [(pos >> (4 * s)) & 15 for s in range(9)]
    assert sorted(slot) == list(range(9)) and 0 <= gap <= 9
    off = {(a, b): 4 * slot[3 * (b // 2) + a // 2] + (2 if slot[3 * (b // 2) + a // 2] >= gap else 0)
           + 2 * (b % 2) + (a % 2) for a in range(6) for b in range(6)}
    used = sorted(off.values())
    assert len(set(used)) == 36 and max(used) < 38
    pad = sorted(set(range(38)) - set(used))
    assert pad[0] % 2 == 0 and pad[1] == pad[0] + 1
    for (a, b), o in off.items():
        if a % 2 == 0:
            assert off[(a + 1, b)] == o + 1 and o % 2 == 0
