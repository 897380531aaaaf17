# SPDX-License-Identifier: Apache-2.0
"""Index schedules of the tensor-core Jacobi (csrc/asg_jacobi_tc.cu), replayed
in Python: the odd-even pair-solve ordering must pair every two indices
exactly once per PW rounds (the cyclic-sweep property of the reference's
sym_eig, densela.hpp:204-246), with the kernel's exact position arithmetic,
its swap rule, and its lane layout of the register-resident rotation."""
import itertools

import pytest


def odd_even_rounds(pw):
    """Positions -> indices over the PW rounds of tj_pair_kernel's odd-even
    pass: round r pairs positions (2k + r%2, 2k + 1 + r%2); the wrap pair
    (PW-1, 0) of odd rounds is the identity without swap; every real pair
    swaps its two positions after rotating."""
    at = list(range(pw))  # index held at each position
    met = []
    for r in range(pw):
        odd = r & 1
        for k in range(pw // 2):
            wrap = odd and k == pw // 2 - 1
            a = 2 * k + odd
            c = 0 if wrap else a + 1
            if wrap:
                continue
            met.append(frozenset((at[a], at[c])))
            at[a], at[c] = at[c], at[a]
    return met, at


@pytest.mark.parametrize("pw", [64, 128])
def test_odd_even_meets_every_pair_once(pw):
    met, final = odd_even_rounds(pw)
    assert len(met) == pw * (pw - 1) // 2
    assert set(met) == {frozenset(p) for p in itertools.combinations(range(pw), 2)}
    assert final == list(reversed(range(pw)))  # odd-even transposition of a reversed sequence


@pytest.mark.parametrize("pw,nt", [(128, 512), (64, 256)])
def test_s_block_mapping_partitions_the_matrix(pw, nt):
    """Every element of S belongs to exactly one 2x2 block in every round."""
    for odd in (0, 1):
        seen = set()
        for e in range((pw // 2) ** 2):
            ki, kj = divmod(e, pw // 2)
            ai = 2 * ki + odd
            bi = 0 if (odd and ki == pw // 2 - 1) else ai + 1
            aj = 2 * kj + odd
            bj = 0 if (odd and kj == pw // 2 - 1) else aj + 1
            for x in ((ai, aj), (ai, bj), (bi, aj), (bi, bj)):
                assert x not in seen
                seen.add(x)
        assert len(seen) == pw * pw


@pytest.mark.parametrize("pw,nt", [(128, 512), (64, 256)])
def test_shared_bank_pattern_is_conflict_free(pw, nt):
    """Half-warps take the two rows in opposite order (row stride PW+1), so
    the 32 lanes of an S load touch 32 distinct banks (except the wrap lane)."""
    ld = pw + 1
    for odd in (0, 1):
        for w in range(nt // 32):
            e0 = w * 32
            for first in (True, False):
                banks = []
                for lane in range(32):
                    e = e0 + lane
                    ki, kj = divmod(e % ((pw // 2) ** 2), pw // 2)
                    ai = 2 * ki + odd
                    bi = 0 if (odd and ki == pw // 2 - 1) else ai + 1
                    aj = 2 * kj + odd
                    flip = bool(lane & 16)
                    row = (bi if flip else ai) if first else (ai if flip else bi)
                    banks.append((row * ld + aj) % 32)
                wrap_lanes = 1 if odd else 0
                assert len(set(banks)) >= 32 - 2 * wrap_lanes


def test_register_z_layout_matches_positions():
    """Wide pairs: warp w owns rows [8w, 8w+8), lane l columns [4l, 4l+4).
    Even rounds pair columns inside a lane; odd rounds pair (4l+1, 4l+2)
    inside and (4l+3, 4l+4) across lanes l, l+1 (lane 31's is the wrap)."""
    pw, cpl = 128, 4
    for odd in (0, 1):
        pairs = set()
        for lane in range(32):
            z0 = lane * cpl
            if not odd:
                for j in range(0, cpl, 2):
                    pairs.add((z0 + j, z0 + j + 1))
            else:
                for j in range(1, cpl - 1, 2):
                    pairs.add((z0 + j, z0 + j + 1))
                if lane < 31:
                    pairs.add((z0 + cpl - 1, z0 + cpl))
        expect = {(2 * k + odd, 2 * k + 1 + odd) for k in range(pw // 2) if not (odd and k == pw // 2 - 1)}
        assert pairs == expect
