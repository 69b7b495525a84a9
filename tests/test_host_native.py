"""libadask host-side bookkeeping (no GPU needed): SeedSequence, PCG64
seeding / jump-ahead / buffered 32-bit draws, Lemire bounded integers,
choice(replace=False) -- against numpy 2.3.5 and the reference golden draws."""
import ctypes as C
import os
import sys

import numpy as np
import pytest

from paper_2104_14101_b200 import _lib
from paper_2104_14101_b200.embeddings import derive_seed, padded_rows

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import recipes as R  # noqa: E402

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden.npz"))
L = _lib.lib()


def test_derive_seed_matches_reference_golden():
    for (b, k), v in zip(G["derive_in"], G["derive_out"]):
        assert derive_seed(int(b), int(k)) == int(v)
        if int(b) < 2**64:
            assert L.adask_derive_seed(int(b), int(k)) == int(v)


@pytest.mark.parametrize("seed", [0, 1, 9, 2**64 - 1, 2**70 + 3, (5, 6), 123456789012345])
def test_pcg64_seeding_matches_numpy(seed):
    g = _lib.pcg64_from_seed(seed)
    st = np.random.PCG64(seed).state["state"]
    assert (g.state_hi << 64 | g.state_lo) == st["state"]
    assert (g.inc_hi << 64 | g.inc_lo) == st["inc"]


@pytest.mark.parametrize("m", [1, 2, 3, 64, 1000, 65536, 2**31 + 1, 3000000007])
def test_bounded_integers_match_numpy(m):
    ref = np.random.default_rng(11).integers(0, m, size=3001)
    g = _lib.pcg64_from_seed(11)
    out = (C.c_int64 * 3001)()
    assert L.adask_pcg64_integers_host(C.byref(g), m, 3001, out) == 0
    assert np.array_equal(np.frombuffer(out, dtype=np.int64), ref)


@pytest.mark.parametrize("i", range(len(R.SRHT_CASES)))
def test_srht_draws_match_reference(i):
    n, d, m, seed = R.SRHT_CASES[i]
    g = _lib.pcg64_from_seed(seed)
    bits = (C.c_int64 * n)()
    L.adask_pcg64_integers_host(C.byref(g), 2, n, bits)
    assert np.array_equal(np.frombuffer(bits, dtype=np.int64), G[f"srht{i}_bits"])
    idx = (C.c_int64 * m)()
    assert L.adask_choice_noreplace(C.byref(g), padded_rows(n), m, idx) == 0
    assert np.array_equal(np.frombuffer(idx, dtype=np.int64), G[f"srht{i}_idx"])
    # the jump-ahead path the SRHT uses (skip n draws, then choice)
    g2 = _lib.pcg64_from_seed(seed)
    L.adask_pcg64_skip_u32(C.byref(g2), n)
    idx2 = (C.c_int64 * m)()
    L.adask_choice_noreplace(C.byref(g2), padded_rows(n), m, idx2)
    assert np.array_equal(np.frombuffer(idx2, dtype=np.int64), G[f"srht{i}_idx"])


@pytest.mark.parametrize("i", range(len(R.SJLT_CASES)))
def test_sjlt_draws_match_reference(i):
    n, d, m, seed = R.SJLT_CASES[i]
    g = _lib.pcg64_from_seed(seed)
    rows = (C.c_int64 * n)()
    L.adask_pcg64_integers_host(C.byref(g), m, n, rows)
    bits = (C.c_int64 * n)()
    L.adask_pcg64_integers_host(C.byref(g), 2, n, bits)
    assert np.array_equal(np.frombuffer(rows, dtype=np.int64), G[f"sjlt{i}_rows"])
    assert np.array_equal(np.frombuffer(bits, dtype=np.int64), G[f"sjlt{i}_bits"])


@pytest.mark.parametrize("N,m", [(64, 16), (10000, 10000), (20001, 400), (20001, 401), (1 << 15, 655),
                                 (1 << 15, 656), (65536, 4096), (1, 1), (5, 0)])
def test_choice_both_branches(N, m):
    rng = np.random.default_rng(3)
    rng.integers(0, 2, size=7)  # odd number of prior draws: buffered half in play
    ref = rng.choice(N, size=m, replace=False)
    g = _lib.pcg64_from_seed(3)
    L.adask_pcg64_skip_u32(C.byref(g), 7)
    out = (C.c_int64 * max(m, 1))()
    assert L.adask_choice_noreplace(C.byref(g), N, m, out) == 0
    assert np.array_equal(np.frombuffer(out, dtype=np.int64)[:m], ref)


def test_sjlt_rows_s_gt_1_and_draw_count():
    n, m, s, seed = 300, 16, 3, 25
    rng = np.random.default_rng(seed)
    ref = np.concatenate([rng.choice(m, size=s, replace=False) for _ in range(n)])
    signs = rng.integers(0, 2, size=n * s)
    g = _lib.pcg64_from_seed(seed)
    rows = np.empty(n * s, dtype=np.int64)
    draws = C.c_uint64()
    assert L.adask_sjlt_rows(C.byref(g), n, m, s, rows.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(draws)) == 0
    assert np.array_equal(rows, ref)
    g2 = _lib.pcg64_from_seed(seed)
    L.adask_pcg64_skip_u32(C.byref(g2), draws.value)
    out = (C.c_int64 * (n * s))()
    L.adask_pcg64_integers_host(C.byref(g2), 2, n * s, out)
    assert np.array_equal(np.frombuffer(out, dtype=np.int64), signs)


def test_philox_gaussian_host_matches_oracle_definition():
    from oracle import adasketch_oracle as O

    m, n, seed = 5, 37, 123456789012345
    out = np.zeros((m, n))
    assert L.adask_philox_gaussian_host(m, 3, n, seed, out.ctypes.data, n) == 0
    np.testing.assert_allclose(out, O.philox_gaussian(m, n, seed, col0=3), rtol=1e-15, atol=1e-16)
