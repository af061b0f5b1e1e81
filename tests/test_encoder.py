"""Host side of the encoder hand-off (encoder.py): the reference's DCT matrix,
zigzag order and quantiser step, and the accumulation model the device DCT
follows (sequential FMA chains in numpy's einsum_path order), pinned against
the reference's own dct8_blocks / idct8_blocks.  Build container only."""
from fractions import Fraction

import numpy as np
import pytest

import refimpl

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not refimpl.available(), reason="/root/reference not present")]


def test_tables_equal_the_reference():
    refimpl.load()
    from fvv.codec import quant_step
    from fvv.dct import _C, ZIGZAG
    from paper_2112_10603_b200 import encoder as E
    assert np.array_equal(E.DCT, _C) and E.DCT.tobytes() == _C.tobytes()
    assert np.array_equal(E.ZIGZAG, ZIGZAG)
    assert all(E.quant_step(q) == quant_step(q) for q in range(101))


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _chain(a, b):
    acc = 0.0
    for j in range(8):
        acc = _fma(float(a[j]), float(b[j]), acc)
    return acc


def test_dct_accumulation_model_matches_reference():
    """k_enc_blocks' FMA chains == the reference's einsum on this host."""
    refimpl.load()
    from fvv.dct import dct8_blocks, idct8_blocks
    from paper_2112_10603_b200.encoder import DCT as C
    rng = np.random.default_rng(5)
    blocks = rng.integers(-255, 256, (12, 8, 8)).astype(np.float64)
    ref = dct8_blocks(blocks)
    q = rng.integers(-40, 41, (12, 8, 8)).astype(np.float64) * 13
    iref = idct8_blocks(q)
    for n in range(blocks.shape[0]):
        T = np.array([[_chain(C[i], blocks[n][:, k]) for k in range(8)] for i in range(8)])
        O = np.array([[_chain(T[i], C[l]) for l in range(8)] for i in range(8)])
        assert np.array_equal(O, ref[n])
        T = np.array([[_chain(C[:, i], q[n][:, k]) for k in range(8)] for i in range(8)])
        O = np.array([[_chain(T[i], C[:, l]) for l in range(8)] for i in range(8)])
        assert np.array_equal(O, iref[n])
