"""The device DEFLATE (csrc/deflate_kernels.cu) against zlib.compress(x, 6)[2:-4],
byte for byte, for every block type and window situation zlib has: empty and
tiny streams, incompressible data (stored blocks, including ones whose start
slid out of the window), static and dynamic blocks, 258-byte runs, window
slides, the end-of-input slide that turns a MAX_DIST candidate into NIL,
16383-symbol block boundaries, token-like streams, and a fuzz batch -- all in
one batched call, as the encoder issues it."""
import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(2024)
    rnd = lambda n, a=256: rng.integers(0, a, n, dtype=np.uint8).tobytes()  # noqa: E731
    cases = [b"", b"a", b"ab", b"abc", b"abcd", rnd(5), rnd(100), bytes(1000), bytes(300000), rnd(70000),
             rnd(200000, 4), rnd(200000, 16), rnd(1000000, 3)]
    text = b"".join(b"the quick brown fox jumps over the lazy dog %d\n" % rng.integers(1000) for _ in range(11000))
    cases.append(text)
    runs = np.where(rng.random(600000) < 0.6, 0, rng.integers(0, 7, 600000)).astype(np.uint8)
    lv = np.where(rng.random(600000) < 0.7, rng.integers(-1, 2, 600000), rng.integers(-20, 21, 600000))
    tok = np.stack([runs, (lv & 0xff).astype(np.uint8), ((lv >> 8) & 0xff).astype(np.uint8)], 1).tobytes()
    cases.append(tok)
    for k in range(3):  # end-of-input slide: candidate at exactly MAX_DIST from strstart = 65274 + 32768 k
        for d in (0, 262, 300):
            n = 65535 + 32768 * k - d + 262
            v = bytearray(rnd(n, 200))
            p = 65274 + 32768 * k
            for j in range(6):
                if p + j < n:
                    v[p + j] = v[p - 32506 + j] = 250 + j
            cases.append(bytes(v))
    for n in (65535, 65536, 65537, 65274, 65275, 98042, 98043, 131072):
        cases.append(rnd(n, 8))
    periodic = bytes(((i % 37) * 7 + i // 5000) & 0xff for i in range(400000))
    cases.append(periodic)
    for _ in range(24):
        parts, total = [], int(rng.integers(1, 300000))
        size = 0
        while size < total:
            kind, ln = int(rng.integers(5)), int(rng.integers(1, 40000))
            if kind == 0:
                seg = rnd(ln)
            elif kind == 1:
                seg = rnd(ln, int(rng.integers(2, 8)))
            elif kind == 2:
                seg = bytes([int(rng.integers(256))]) * ln
            else:
                seg = bytes((i % int(rng.integers(1, 300))) & 0xff for i in range(ln))
            parts.append(seg)
            size += ln
        cases.append(b"".join(parts)[:total])
    return cases


def test_device_deflate_matches_zlib():
    import torch
    from paper_2112_10603_b200.deflate import deflate_bytes
    cases = _cases()
    offs = np.concatenate([[0], np.cumsum([len(c) for c in cases])]).tolist()
    data = torch.frombuffer(bytearray(b"".join(cases)), dtype=torch.uint8).cuda()
    got = deflate_bytes(data, offs)
    bad = []
    for i, (c, g) in enumerate(zip(cases, got)):
        ref = zlib.compress(c, 6)[2:-4]
        if g != ref:
            j = next((k for k in range(min(len(g), len(ref))) if g[k] != ref[k]), min(len(g), len(ref)))
            bad.append(f"case {i} (n={len(c)}): {len(g)} vs {len(ref)} bytes, first difference at {j}")
    assert not bad, "\n".join(bad)


def test_device_deflate_single_and_offset_streams():
    """A stream that does not start at the buffer's beginning, alone in its batch."""
    import torch
    from paper_2112_10603_b200.deflate import deflate_bytes
    rng = np.random.default_rng(5)
    buf = rng.integers(0, 6, 250007, dtype=np.uint8).tobytes()
    data = torch.frombuffer(bytearray(buf), dtype=torch.uint8).cuda()
    got = deflate_bytes(data, [13, 250007])
    assert got[0] == zlib.compress(buf[13:], 6)[2:-4]
