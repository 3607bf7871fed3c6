"""Search / check the consumer lane permutation of the pull SpMV (csrc/pcg.cu,
kPullUnitOfLane).

Model (sm_100a shared memory): a warp's 16-byte load is served in quarter-warp phases
of 8 lanes; a phase costs as many wavefronts as the largest number of its lanes that
hit the same 16-byte bank group (word index mod 8).  Consumer lane L computes unit
u = 3 j + h (block j of the node's slot, output pair h).  A record holds the 6x6 block as
nine 2x2 sub-blocks (A, B) of 4 doubles (column-major inside) at word SUBW[3 B + A]; per
instruction t = 0..5 (sub-block sb = t / 2, 16-byte half t % 2) the unit reads
  own block j (< 5):    word OWN + 19 (b_i + j) + SUBW[3 sb + h] + t % 2   (sub-blocks (h, sb))
  pulled block j (>= 5): word 80 i + 19 (j - 5) + SUBW[3 h + sb] + t % 2    (sub-blocks (sb, h))
with the 38-double record stride (19 words), the 80-word pulled slot per node and the
own region after the pulled slots (OWN = 80 C), i = node index in the chunk, b_i = 5 i
(interior nodes).  The row-pair store red[27 e + u] is modelled too.  A second term
keeps the three lanes of a block (same 48-byte x gather) in one quarter warp.

    python tools/pull_lane_perm.py            # check the table in pcg.cu
    python tools/pull_lane_perm.py --search   # search a new one
"""
import random
import re
import sys
from pathlib import Path

UNITS = [(j, h) for j in range(9) for h in range(3)]
C = 12  # nodes per chunk (default variant)


def sub_words():
    """word offset of each sub-block 3 B + A inside a record (csrc/sso_internal.h
    PULL_SUB_POS / PULL_SUB_GAP: slot q at word 2 q, + 1 from the pad word on)."""
    src = (Path(__file__).resolve().parents[1] / "paper_2407_20026_b200" / "csrc" / "sso_internal.h").read_text()
    pos = int(re.search(r"PULL_SUB_POS = (0x[0-9a-f]+)ull", src).group(1), 16)
    gap = int(re.search(r"PULL_SUB_GAP = (\d+);", src).group(1))
    slots = [(pos >> (4 * s)) & 15 for s in range(9)]
    return [2 * q + (1 if q >= gap else 0) for q in slots]


SUBW = sub_words()


def words(j, h, t, i, bi):
    sb, half = t // 2, t % 2  # 2x2 sub-block index along the unit's strip, which 16-byte half
    if j < 5:   # own K_mj: sub-blocks (A, B) = (h, sb)
        return 80 * C + 19 * (bi + j) + SUBW[3 * sb + h] + half
    return 80 * i + 19 * (j - 5) + SUBW[3 * h + sb] + half  # pulled: sub-blocks (sb, h)


def phases(ws):
    tot = 0
    for q in range(4):
        cnt = {}
        for w in ws[8 * q:8 * q + 8]:
            if w is not None:
                cnt[w % 8] = cnt.get(w % 8, 0) + 1
        tot += max(cnt.values()) if cnt else 0
    return tot


def wavefronts(perm, nodes=None):
    """Mean wavefronts per 16-byte shared instruction (6 loads + 1 store per node)."""
    nodes = nodes or [(i, 5 * i) for i in range(C)]
    tot = 0
    for i, bi in nodes:
        for t in range(6):
            tot += phases([None if u is None else words(*UNITS[u], t, i, bi) for u in perm])
        tot += phases([None if u is None else 27 * (i // 4) + u for u in perm])
    return tot / len(nodes) / 7


def split_blocks(perm):
    return sum(len({L // 8 for L, u in enumerate(perm) if u is not None and UNITS[u][0] == j}) - 1
               for j in range(9))


def table_from_source():
    src = (Path(__file__).resolve().parents[1] / "paper_2407_20026_b200" / "csrc" / "pcg.cu").read_text()
    m = re.search(r"kPullUnitOfLane\[32\]\s*=\s*\{([^}]*)\}", src)
    vals = [int(v) for v in m.group(1).replace("\n", " ").split(",")]
    return [None if v >= 27 else v for v in vals]


def search(seeds=8, iters=40000):
    base = list(range(27)) + [None] * 5
    best, bc = None, 1e9
    for seed in range(seeds):
        random.seed(seed)
        cur = base[:]
        random.shuffle(cur)
        cc = wavefronts(cur) + 0.25 * split_blocks(cur)
        for _ in range(iters):
            a, c = random.sample(range(32), 2)
            cand = cur[:]
            cand[a], cand[c] = cand[c], cand[a]
            x = wavefronts(cand) + 0.25 * split_blocks(cand)
            if x <= cc:
                cur, cc = cand, x
        if cc < bc:
            best, bc = cur, cc
    return best


if __name__ == "__main__":
    if "--search" in sys.argv:
        p = search()
        print([31 if u is None else u for u in p], wavefronts(p), split_blocks(p))
    else:
        p = table_from_source()
        print("identity:", wavefronts(list(range(27)) + [None] * 5))
        print("table:   ", wavefronts(p), "wavefronts per instruction,", split_blocks(p), "split block(s)")

