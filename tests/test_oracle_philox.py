"""Pins of the oracle's Philox4x32-10 and Bernoulli mask (Eq.2).

- Library routine: NVIDIA curand_Philox4x32_10 (compiled for the host from
  /usr/local/cuda/include/curand_philox4x32_x.h) on 2e5 random (ctr, key) pairs,
  bit-exact.
- p = 1 selects every code (M^t = identity).
- Bernoulli(p) statistics: popcount within 6 sigma of Binomial(K*Hc*Wc, p);
  masks of different iterations overlap at rate ~p^2 ("a different matrix M^t"
  per iteration); same (seed, t) is deterministic.
"""
import os
import shutil
import struct
import subprocess
import tempfile

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def curand_ref():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    out = os.path.join(tempfile.mkdtemp(prefix="curand_ref_"), "curand_ref")
    subprocess.run([nvcc, "-O2", "-Wno-deprecated-gpu-targets", "-o", out,
                    os.path.join(HERE, "helpers", "curand_philox_ref.cu")], check=True)
    return out


def _run_curand(exe, ctr, key):
    count = ctr.shape[0]
    payload = struct.pack("<Q", count) + np.concatenate([ctr, key], axis=1).astype("<u4").tobytes()
    res = subprocess.run([exe], input=payload, stdout=subprocess.PIPE, check=True)
    return np.frombuffer(res.stdout, dtype="<u4").reshape(count, 4)


def test_philox_matches_curand(curand_ref):
    rng = np.random.default_rng(12345)
    n = 200_000
    ctr = rng.integers(0, 2**32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    # edge counters: zeros, all-ones, the mask counter form {q lo, q hi, t, tag}
    ctr[0] = 0; key[0] = 0
    ctr[1] = 0xFFFFFFFF; key[1] = 0xFFFFFFFF
    ctr[2] = [7, 0, 3, 0x4353434D]; key[2] = [0xDEADBEEF, 0x12345678]
    ref = _run_curand(curand_ref, ctr, key)
    got = oracle.philox4x32_10(ctr, key)
    assert np.array_equal(got, ref)


def test_mask_bits_layout_against_curand(curand_ref):
    """Bit l = (k*Hc+u)*Wc+v of word l>>5 is curand(ctr={q lo,q hi,t,tag}, key=seed)[l&3] < floor(p*2^32)."""
    K, Hc, Wc, p, seed, t = 3, 7, 9, 0.37, 0x0123456789ABCDEF, 5
    bits = oracle.mask_bits(K, Hc, Wc, p, seed, t)
    m = oracle.unpack_mask(bits, K, Hc, Wc).ravel()
    L = K * Hc * Wc
    q = np.arange((L + 3) // 4, dtype=np.uint64)
    ctr = np.stack([q & 0xFFFFFFFF, q >> 32, np.full_like(q, t), np.full_like(q, 0x4353434D)],
                   axis=1).astype(np.uint32)
    key = np.tile(np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint64), (len(q), 1)).astype(np.uint32)
    w = _run_curand(curand_ref, ctr, key).ravel()[:L]
    thr = int(np.floor(p * 2.0 ** 32))
    assert np.array_equal(m, w.astype(np.uint64) < thr)
    # padding bits beyond K*Hc*Wc are zero
    allbits = np.unpackbits(bits.view(np.uint8), bitorder="little")
    assert not allbits[L:].any()


def test_mask_p1_is_identity():
    K, Hc, Wc = 4, 13, 11
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, 1.0, 99, 3), K, Hc, Wc)
    assert m.all()
    assert oracle.mask_threshold(1.0) == 2 ** 32


@pytest.mark.parametrize("p", [0.05, 0.1, 0.5])
def test_mask_bernoulli_statistics(p):
    K, Hc, Wc = 8, 64, 64
    n = K * Hc * Wc
    m1 = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, 2024, 1), K, Hc, Wc)
    m2 = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, 2024, 2), K, Hc, Wc)
    sd = np.sqrt(n * p * (1 - p))
    for m in (m1, m2):
        assert abs(int(m.sum()) - n * p) < 6 * sd
    ov = int((m1 & m2).sum())
    sd2 = np.sqrt(n * p * p * (1 - p * p))
    assert abs(ov - n * p * p) < 6 * sd2
    # determinism
    m1b = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, 2024, 1), K, Hc, Wc)
    assert np.array_equal(m1, m1b)
    # different seeds differ
    m3 = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, 2025, 1), K, Hc, Wc)
    assert not np.array_equal(m1, m3)


def test_mask_threshold_rounding():
    assert oracle.mask_threshold(0.5) == 2 ** 31
    assert oracle.mask_threshold(0.1) == int(np.floor(0.1 * 2.0 ** 32))
    assert oracle.mask_threshold(2.0 ** -32) == 1


# ---- block-structured masks (reading E5)
SECTOR_TAG = 0x43534253


def test_sector8_mask_layout_against_curand(curand_ref):
    """Bit l is curand(ctr={q lo, q hi, t, tag'}, key=seed)[b & 3] < thr with b = l >> 3, q = b >> 2:
    one draw per aligned block of 8 coordinates, blocks running across plane boundaries."""
    K, Hc, Wc, p, seed, t = 3, 7, 9, 0.37, 0x0123456789ABCDEF, 5
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, seed, t, mode="sector8"), K, Hc, Wc).ravel()
    L = K * Hc * Wc
    nb = (L + 7) // 8
    q = np.arange((nb + 3) // 4, dtype=np.uint64)
    ctr = np.stack([q & 0xFFFFFFFF, q >> 32, np.full_like(q, t), np.full_like(q, SECTOR_TAG)],
                   axis=1).astype(np.uint32)
    key = np.tile(np.array([seed & 0xFFFFFFFF, seed >> 32], dtype=np.uint64), (len(q), 1)).astype(np.uint32)
    w = _run_curand(curand_ref, ctr, key).ravel()[:nb]
    thr = int(np.floor(p * 2.0 ** 32))
    expect = np.repeat(w.astype(np.uint64) < thr, 8)[:L]
    assert np.array_equal(m, expect)


@pytest.mark.parametrize("p", [0.1, 0.5])
def test_sector8_mask_blocks_and_statistics(p):
    K, Hc, Wc = 8, 64, 64
    n = K * Hc * Wc
    m = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, p, 77, 3, mode="sector8"), K, Hc, Wc).ravel()
    blocks = m.reshape(-1, 8)
    assert (blocks.all(axis=1) | ~blocks.any(axis=1)).all()  # constant on every aligned block
    nbk = n // 8
    sd = np.sqrt(nbk * p * (1 - p))
    assert abs(int(blocks[:, 0].sum()) - nbk * p) < 6 * sd
    full = oracle.unpack_mask(oracle.mask_bits(K, Hc, Wc, 1.0, 77, 3, mode="sector8"), K, Hc, Wc)
    assert full.all()
