"""Host-side checks of the shared-memory layouts the last kernels rely on (no GPU):

* the warp-per-pair K1 (csrc/k_time.cuh k_time_wp): the lane -> partner-job table kWpPj is a
  permutation, every stage's scratch layout is a bijection of the 256 positions into the warp's
  WSLOTS slots that the matching read finds again, and each 8-lane phase of every access hits
  eight distinct 16-byte bank groups (conflict free);
* the transposed strided store (csrc/k_line.cu, k_line TS): the box {a < T-1, q < 2L} holds grid
  row p = 2L a + q at slot q (T-1) + a exactly once, consecutive threads write consecutive slots,
  and the last thread's rows (stored directly) complete the line.
"""
import os
import re

import numpy as np

SRC = os.path.join(os.path.dirname(__file__), "..", "paper_2603_04350_b200", "csrc")


def wp_table():
    txt = open(os.path.join(SRC, "k_time.cuh")).read()
    m = re.search(r"kWpPj\[32\]\s*=\s*\{([^}]*)\}", txt)
    return [int(x) for x in m.group(1).replace("\n", " ").split(",")]


NT, NSL, WS = 256, 64, 256 + 32


def jb_of(ja):
    return NSL // 2 if ja == 0 else NSL - ja


def l8(p):  # one pad per 8 positions (L1, L2, L4)
    return p + (p >> 3)


def l32(p):  # one pad per 32 positions (L3)
    return p + (p >> 5)


def banks_distinct(slots):
    """each 8-lane phase of a warp access (16-byte slots): distinct bank groups"""
    slots = np.asarray(slots)
    return all(len(set((slots[q * 8:(q + 1) * 8] % 8).tolist())) == 8 for q in range(len(slots) // 8))


def test_wp_partner_table_is_a_permutation():
    t = wp_table()
    assert sorted(t) == list(range(32))
    assert sorted(t + [jb_of(x) for x in t]) == list(range(64))  # ja, jb cover every partner job


def test_wp_scratch_layouts_bijective_and_conflict_free():
    lanes = np.arange(32)
    ja = np.array(wp_table())
    jb = np.array([jb_of(x) for x in ja])
    # (writer positions per lane and r, reader positions per lane and r, layout)
    stages = {
        "L1 stage 0 -> middle": ([8 * j + r for r in range(8) for j in lanes], [j + 32 * r for r in range(8) for j in lanes], l8),
        "L2 middle -> partner": ([(j // 8) * 64 + j % 8 + 8 * r for r in range(8) for j in lanes],
                                 [x + 64 * r for r in range(4) for x in np.concatenate([ja, jb])], l8),
        "L3 partner -> inverse middle": ([4 * x + r for r in range(4) for x in np.concatenate([ja, jb])],
                                         [j + 32 * r for r in range(8) for j in lanes], l32),
        "L4 inverse middle -> final": ([(j // 4) * 32 + j % 4 + 4 * r for r in range(8) for j in lanes],
                                       [j + 32 * r for r in range(8) for j in lanes], l8),
    }
    for name, (wr, rd, lay) in stages.items():
        assert sorted(wr) == list(range(NT)), name
        assert sorted(rd) == list(range(NT)), name
        slots = [lay(p) for p in range(NT)]
        assert len(set(slots)) == NT and max(slots) < WS, name
        # every warp instruction (fixed r; the partner accesses once for ja, once for jb)
        for acc in (wr, rd):
            for k in range(0, len(acc), 32):
                assert banks_distinct([lay(p) for p in acc[k:k + 32]]), (name, k)


def test_wp_kernel_uses_these_layouts():
    """the kernel's per-lane bases are the layouts above (guards against an edit of one side)"""
    txt = open(os.path.join(SRC, "k_time.cuh")).read()
    for frag in ("const int l1w = 9 * j;", "const int lrd = j + (j >> 3);", "const int l2w = (j >> 3) * 72 + (j & 7);",
                 "const int l2a = ja + (ja >> 3), l2b = jb + (jb >> 3);",
                 "const int l3a = 4 * ja + (ja >> 3), l3b = 4 * jb + (jb >> 3);",
                 "const int l4w = (j >> 2) * 36 + (j & 3);", "W[l4w + 4 * r + (r >> 1)]", "W[j + 33 * r]"):
        assert frag in txt, frag
    for j in range(32):  # the bases equal the layout functions at r = 0 (and the r strides below)
        assert 9 * j == l8(8 * j) and j + (j >> 3) == l8(j)
        assert (j >> 3) * 72 + (j & 7) == l8((j // 8) * 64 + j % 8)
        assert (j >> 2) * 36 + (j & 3) == l8((j // 4) * 32 + j % 4)
        for r in range(8):
            assert l8(j + 32 * r) == j + (j >> 3) + 36 * r
            assert l8((j // 8) * 64 + j % 8 + 8 * r) == (j >> 3) * 72 + (j & 7) + 9 * r
            assert l32(j + 32 * r) == j + 33 * r
            assert l8((j // 4) * 32 + j % 4 + 4 * r) == (j >> 2) * 36 + (j & 3) + 4 * r + (r >> 1)
    for x in range(64):
        for r in range(4):
            assert l8(x + 64 * r) == x + (x >> 3) + 72 * r
            assert l32(4 * x + r) == 4 * x + (x >> 3) + r


def test_transposed_store_view_covers_the_line_once():
    for M, R0 in ((256, 8), (512, 16), (1024, 16), (2048, 16), (4096, 16)):
        T, L = M // R0, R0 // 2
        seen = {}
        for a in range(T - 1):
            for q in range(2 * L):
                slot = q * (T - 1) + a
                assert slot not in seen
                seen[slot] = 2 * L * a + q
        # the box's smem order is dim a innermost: slot = q (T-1) + a <-> row 2L a + q
        assert sorted(seen.values()) == list(range(2 * L * (T - 1)))
        # the last thread's rows: M - 2L .. M - 2 (M - 1 is the spectral pad)
        tail = [2 * L * (T - 1) + q for q in range(2 * L - 1)]
        assert sorted(list(seen.values()) + tail) == list(range(M - 1))
        # consecutive threads a, a+1 write consecutive 16-byte slots in every instruction q
        for q in range(2 * L):
            s = [q * (T - 1) + a for a in range(min(32, T - 1))]
            assert all(b - a_ == 1 for a_, b in zip(s, s[1:]))
