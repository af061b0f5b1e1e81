"""CPU checks of the rounding arguments the exact kernels rely on.

fvv_device.cuh `third_scaled_f32`: the occlusion cue's column pass is
f32(RN_f64(sn * 2^-k / 3)) in the reference (scipy's f64 running sum of an f32
plane, cast back to f32); the kernels compute it as f32(RN_f64(sn * c3k)) with
c3k = RN(1/3) * 2^-k -- one multiply.  numpy's f64 division is the correctly
rounded quotient, so comparing the two casts over a large sample (every small
sn, multiples of 3, powers of two and their neighbours, random sn < 2^32) checks
the claim at every scale k the geometry can produce.
"""
import numpy as np
import pytest

R3 = float.fromhex("0x1.5555555555555p-2")


def _cases(rng):
    small = np.arange(0, 1 << 16, dtype=np.uint64)
    rnd = rng.integers(0, 1 << 32, 1 << 20, dtype=np.uint64)
    mul3 = rng.integers(0, (1 << 32) // 3, 1 << 18, dtype=np.uint64) * 3
    p2 = np.array([1 << e for e in range(32)], dtype=np.uint64)
    near = np.concatenate([p2 - 1, p2, p2 + 1, 3 * p2[:30], 3 * p2[:30] - 1, 3 * p2[:30] + 1])
    s = np.concatenate([small, rnd, mul3, near])
    return s[s < (1 << 32)]


@pytest.mark.parametrize("k", [1, 8, 12, 15, 16, 17, 20, 24, 30])
def test_single_multiply_third_matches_correctly_rounded(k):
    rng = np.random.default_rng(k)
    sn = _cases(rng).astype(np.float64)            # exact: sn < 2^53
    ref = ((sn * 2.0 ** -k) / 3.0).astype(np.float32)   # RN_f64 quotient, then f32
    c3k = R3 * 2.0 ** -k                           # exact power-of-two scale
    got = (sn * c3k).astype(np.float32)
    bad = np.nonzero(ref != got)[0]
    assert bad.size == 0, f"k={k}: sn={sn[bad[:5]]}"
