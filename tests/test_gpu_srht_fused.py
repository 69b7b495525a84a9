"""The fused SRHT kernel (csrc/srht_fused.cu: both FWHT passes in one
persistent kernel, Z kept in L2) against the reference SRHT (oracle,
embeddings.py:81-102): bit for bit in fp64, and bitwise equal to the
two-launch tile kernels in fp32.  Covers pass-2 widths 1..10 bits, pruned and
identity slot sets, ragged n (zero padding), partial 64-byte panels (odd fp32
widths), strided rows, several column groups, accumulation and repeated
launches (the kernel's self-resetting counters)."""
import numpy as np
import pytest
import torch

from oracle import adasketch_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ak():
    import paper_2104_14101_b200 as ak

    return ak


def _fused(monkeypatch, **env):
    monkeypatch.delenv("ADASK_FWHT_PIPE", raising=False)
    monkeypatch.setenv("ADASK_SRHT_FUSED", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, str(v))


@pytest.mark.parametrize("n,d,m,seed", [
    (512, 16, 40, 1),             # pass 2 = 1 bit
    (2048, 16, 40, 1),            # 3 bits
    (4096, 24, 3000, 2),          # 4 bits, identity slots
    (5024, 9, 700, 3),            # 8192 padded (zero rows), partial panel
    (1 << 15, 20, 1 << 15, 4),    # every padded row selected
    (65536, 40, 32, 5),           # config-1 shape, few slots
    (65536, 40, 4096, 6),         # config-1 shape, all slots
    ((1 << 15) + 32, 17, 513, 7),  # 2^16 padded, zero rows
    ((1 << 16) + 32, 6, 2000, 8),  # past the fused range (2^17): two-launch path
])
def test_fused_srht_bitwise(ak, n, d, m, seed, monkeypatch):
    _fused(monkeypatch)
    A = np.random.default_rng(seed).standard_normal((n, d))
    got = ak.sketch_srht(A, m, seed).SA
    assert np.array_equal(got, O.sketch_srht(A, m, seed))


@pytest.mark.parametrize("zmb,lag", [(1, 1), (2, 2), (1, 5), (1000, 1)])
def test_fused_srht_groups_and_variants(ak, zmb, lag, monkeypatch):
    """Several column groups (Z budget of 1-2 MB: pass 2 of a group overlaps
    pass 1 of later groups, lag 1-5 groups) and a single group."""
    _fused(monkeypatch, ADASK_SRHT_FUSED_ZMB=zmb, ADASK_SRHT_FUSED_LAG=lag)
    A = np.random.default_rng(11).standard_normal((1 << 16, 72))
    for m in (64, 4096):
        assert np.array_equal(ak.sketch_srht(A, m, 3).SA, O.sketch_srht(A, m, 3))


def test_fused_srht_strided_and_repeated(ak, monkeypatch):
    """A column slice (lda > d, 16-byte aligned start, partial last panel), launched three times
    (counters reset by each launch's last CTA)."""
    from paper_2104_14101_b200.embeddings import srht_dev

    _fused(monkeypatch, ADASK_SRHT_FUSED_ZMB=1)
    full = np.random.default_rng(4).standard_normal((1 << 15, 64))
    Ad = torch.from_numpy(full).cuda()[:, 6:43]
    ref = O.sketch_srht(full[:, 6:43], 1500, 8)
    for _ in range(3):
        assert np.array_equal(srht_dev(Ad, 1500, 8).cpu().numpy(), ref)


@pytest.mark.parametrize("n,d,m", [(1 << 16, 64, 64), (1 << 16, 37, 4096), ((1 << 16) - 64, 16, 3000),
                                   (3008, 5, 100)])
def test_fused_srht_fp32_matches_tile_kernels(ak, n, d, m, monkeypatch):
    """fp32 (packed pairs; odd widths end in a half lane): bitwise the tile
    kernels' result, and within fp32 rounding of the fp64 oracle."""
    from paper_2104_14101_b200.embeddings import srht_dev

    A = torch.randn(n, d, dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(n + m))
    _fused(monkeypatch)
    fused = srht_dev(A, m, 9)
    monkeypatch.setenv("ADASK_FWHT_PIPE", "0")
    tile = srht_dev(A, m, 9)
    assert torch.equal(fused, tile)
    ref = O.sketch_srht(A.double().cpu().numpy(), m, 9)
    assert np.linalg.norm(fused.double().cpu().numpy() - ref) <= 1e-5 * np.linalg.norm(ref)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_fused_srht_accumulate(ak, dtype, monkeypatch):
    """out += SRHT (the block-SRHT accumulation of a row-sharded sketch):
    bitwise the tile kernels' accumulation."""
    from paper_2104_14101_b200.embeddings import srht_dev

    A = torch.randn(20000 + 32 * 3, 24, dtype=dtype, device="cuda", generator=torch.Generator("cuda").manual_seed(3))
    base = torch.randn(900, 24, dtype=dtype, device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    _fused(monkeypatch)
    o1 = base.clone()
    srht_dev(A, 900, 21, out=o1, accumulate=True)
    monkeypatch.setenv("ADASK_FWHT_PIPE", "0")
    o2 = base.clone()
    srht_dev(A, 900, 21, out=o2, accumulate=True)
    assert torch.equal(o1, o2)


# ---- blocks of 2^19 .. 2^22 padded rows: the fused kernel per 2^18-row
# sub-block + the combine of the partials (srht_fused_big)
@pytest.mark.parametrize("n,d,m,seed", [
    (1 << 19, 6, 300, 1),               # two sub-blocks
    ((1 << 19) + 32, 5, 2000, 2),       # 2^20 padded: sub-block 2 has 32 rows, sub-block 3 none
    ((1 << 20) - 4096, 4, 70000, 3),    # four sub-blocks, repeated low parts, ragged tail
    (1 << 21, 2, 64, 4),                # config-4 block length, eight sub-blocks
])
def test_fused_srht_big_blocks_bitwise(ak, n, d, m, seed, monkeypatch):
    _fused(monkeypatch)
    A = np.random.default_rng(seed).standard_normal((n, d))
    got = ak.sketch_srht(A, m, seed).SA
    assert np.array_equal(got, O.sketch_srht(A, m, seed))


@pytest.mark.parametrize("n,d,m,acc", [(1 << 19, 24, 1000, False), ((1 << 20) + 64, 9, 5000, True),
                                       (1 << 22, 4, 300, False)])
def test_fused_srht_big_blocks_fp32_match_two_launch(ak, n, d, m, acc, monkeypatch):
    """fp32, incl. accumulation into an existing sketch (the block SRHT of
    config 4 adds its blocks' sketches) and sixteen sub-blocks: bitwise the
    two-launch pipeline's result."""
    from paper_2104_14101_b200.embeddings import srht_dev

    A = torch.randn(n, d, dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(n + m))
    base = torch.randn(m, d, dtype=torch.float32, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    _fused(monkeypatch)
    got = srht_dev(A, m, 5, out=base.clone(), accumulate=True) if acc else srht_dev(A, m, 5)
    monkeypatch.setenv("ADASK_SRHT_FUSED", "0")
    ref = srht_dev(A, m, 5, out=base.clone(), accumulate=True) if acc else srht_dev(A, m, 5)
    assert torch.equal(got, ref)
