"""CPU checks of the VINet path: the fp32 oracle's building blocks and the
packed-weight contract of the tensor-core convolution (include/fvv_b200.h),
emulated as the same GEMM on the CPU."""
import numpy as np
import torch
import torch.nn.functional as Fn

from oracle import vinet_ref as V
from paper_2112_10603_b200 import convtc
from paper_2112_10603_b200.vinet_params import LAYERS, make_params


def test_oracle_primitives():
    g = torch.Generator().manual_seed(0)
    img = torch.rand((3, 12, 20), generator=g)
    z = torch.zeros((12, 20))
    assert torch.equal(V.warp(img, z, z), img)
    c = torch.full((2, 5, 7), 3.25)
    assert torch.equal(V.up2(c), torch.full((2, 10, 14), 3.25))
    x = torch.arange(16.0).reshape(1, 4, 4)
    assert torch.equal(V.pool2(x), torch.tensor([[[2.5, 4.5], [10.5, 12.5]]]))
    # integer shift: warp by (+1, 0) reads the right neighbour (clamped at the edge)
    fx = torch.ones((12, 20))
    w = V.warp(img, fx, z)
    assert torch.allclose(w[:, :, :-1], img[:, :, 1:]) and torch.allclose(w[:, :, -1], img[:, :, -1])


def test_params_deterministic():
    a, b = make_params(3), make_params(3)
    assert len(a) == 3 and all(len(x) == len(LAYERS) for x in a)
    for x, y in zip(a, b):
        for (wa, ba), (wb, bb) in zip(x, y):
            assert torch.equal(wa, wb) and torch.equal(ba, bb)


def _gemm_conv(x_nhwc, wp, cout, k, s, p, taps, base, grid, om, oa, out_shape):
    """The kernel's GEMM: out[g*om + oa] = sum_t x[g*s + base + tap_t] . wp[:, t*cpad:(t+1)*cpad]."""
    B, H, W, cp = x_nhwc.shape
    Hg, Wg = grid
    out = torch.zeros(out_shape)
    xp = x_nhwc.float()
    for gy in range(Hg):
        for gx in range(Wg):
            acc = torch.zeros((B, wp.shape[0]))
            for t, (dy, dx) in enumerate(taps):
                iy, ix = gy * s + base + dy, gx * s + base + dx
                if 0 <= iy < H and 0 <= ix < W:
                    acc += xp[:, iy, ix, :] @ wp[:, t * cp:(t + 1) * cp].float().t()
            out[:, gy * om + oa[0], gx * om + oa[1], :] = acc[:, :cout]
    return out


def test_pack_conv_layout():
    g = torch.Generator().manual_seed(1)
    cin, cout, H, W = 6, 24, 7, 9
    x = torch.randn((1, cin, H, W), generator=g).to(torch.bfloat16).float()
    w = torch.randn((cout, cin, 3, 3), generator=g).to(torch.bfloat16).float()
    cp, nt = convtc.cpad_of(cin), convtc.ntile_of(cout)
    wp = convtc.pack_conv(w, cp, nt)
    assert wp.shape == (nt, 9 * cp)
    xn = torch.zeros((1, H, W, cp))
    xn[..., :cin] = x.permute(0, 2, 3, 1)
    for s in (1, 2):
        ref = Fn.conv2d(x, w, stride=s, padding=1).permute(0, 2, 3, 1)
        Ho, Wo = ref.shape[1:3]
        taps = [(t // 3, t % 3) for t in range(9)]
        got = _gemm_conv(xn, wp, cout, 3, s, 1, taps, -1, (Ho, Wo), 1, (0, 0), (1, Ho, Wo, cout))
        assert torch.allclose(got, ref, atol=1e-4, rtol=1e-4)


def test_pack_convT_layout():
    g = torch.Generator().manual_seed(2)
    cin, cout, H, W = 16, 5, 4, 6
    x = torch.randn((1, cin, H, W), generator=g).to(torch.bfloat16).float()
    w = torch.randn((cin, cout, 4, 4), generator=g).to(torch.bfloat16).float()
    cp, nt = convtc.cpad_of(cin), convtc.ntile_of(cout)
    wp = convtc.pack_convT(w, cp, nt)
    assert wp.shape == (4, nt, 4 * cp)
    ref = Fn.conv_transpose2d(x, w, stride=2, padding=1).permute(0, 2, 3, 1)
    xn = torch.zeros((1, H, W, cp))
    xn[..., :cin] = x.permute(0, 2, 3, 1)
    off = {0: (0, -1), 1: (1, 0)}  # include/fvv_b200.h: input offsets per output parity
    got = torch.zeros((1, 2 * H, 2 * W, cout))
    for ph in range(4):
        a, b = ph >> 1, ph & 1
        taps = [(off[a][t >> 1], off[b][t & 1]) for t in range(4)]
        got += _gemm_conv(xn, wp[ph], cout, 4, 1, 0, taps, 0, (H, W), 2, (a, b), (1, 2 * H, 2 * W, cout))
    assert torch.allclose(got, ref, atol=1e-4, rtol=1e-4)


def test_oracle_flows_small():
    P = make_params(0)
    w, h = 64, 64
    rng = np.random.default_rng(0)
    a = rng.integers(0, 256, w * h * 3 // 2, dtype=np.uint8)
    st = V.flows(a, a, w, h, 1, P)
    assert st.shape == (5, h, w) and torch.isfinite(st).all()
    v = V.synth(a, a, w, h, 1, st, 0.5)
    assert v.shape == a.shape


def test_pack_convT_subpixel_layout():
    """ConvTranspose2d(k4 s2 p1) == one 3x3 conv with 4*Cout sub-pixel outputs (the u1 head)."""
    g = torch.Generator().manual_seed(3)
    cin, cout, H, W = 16, 5, 4, 6
    x = torch.randn((1, cin, H, W), generator=g).to(torch.bfloat16).float()
    w = torch.randn((cin, cout, 4, 4), generator=g).to(torch.bfloat16).float()
    cp = convtc.cpad_of(cin)
    wp = convtc.pack_convT_subpixel(w, cp, 32)
    assert wp.shape == (32, 9 * cp)
    ref = Fn.conv_transpose2d(x, w, stride=2, padding=1).permute(0, 2, 3, 1)
    xn = torch.zeros((1, H, W, cp))
    xn[..., :cin] = x.permute(0, 2, 3, 1)
    taps = [(t // 3, t % 3) for t in range(9)]
    g20 = _gemm_conv(xn, wp, 4 * cout, 3, 1, 1, taps, -1, (H, W), 1, (0, 0), (1, H, W, 4 * cout))
    got = torch.zeros((1, 2 * H, 2 * W, cout))
    for ph in range(4):
        got[:, (ph >> 1)::2, (ph & 1)::2, :] = g20[..., ph * cout:(ph + 1) * cout]
    assert torch.allclose(got, ref, atol=1e-4, rtol=1e-4)
