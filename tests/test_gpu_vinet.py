"""VINet (north-star CNN path) on B200 vs the fp32 torch oracle (oracle/vinet_ref.py).

The convolutions run bf16 x bf16 -> fp32 on tcgen05, so the flows match the
fp32 oracle within a tolerance; the synthesis kernel restates the oracle's
fp32 arithmetic and is checked on the oracle's own flows.
"""
import numpy as np
import pytest

from oracle import vinet_ref as V

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def _pair(w, h, fmt, shift, seed):
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    big = gaussian_filter(rng.random((h + 8, w + 2 * abs(shift) + 8)) * 255.0, 2.5)
    big = (big - big.min()) / (np.ptp(big) + 1e-9) * 230 + 12
    a, b = big[4:4 + h, 4:4 + w], big[4:4 + h, 4 + shift:4 + shift + w]

    def pack(p):
        p = np.rint(p).astype(np.uint8)
        if fmt == 0:
            return p.reshape(-1)
        if fmt == 2:
            return np.stack([p, np.roll(p, 5, 1), 255 - p], -1).reshape(-1)
        cw, ch = w // 2, h // 2
        u = p.reshape(ch, 2, cw, 2).mean((1, 3)).astype(np.uint8)
        return np.concatenate([p.reshape(-1), u.reshape(-1), (255 - u).reshape(-1)])
    return pack(a), pack(b)


CASES = [(448, 256, 2, 3), (256, 192, 1, 4), (192, 128, 0, -2), (200, 124, 1, 5)]  # last: canvas padding


@pytest.fixture(scope="module")
def params():
    from paper_2112_10603_b200.vinet_params import make_params
    return make_params(0)


@pytest.mark.parametrize("w,h,fmt,shift", CASES)
def test_vinet_flows_match_fp32_oracle(torch_cuda, params, w, h, fmt, shift):
    torch = torch_cuda
    from paper_2112_10603_b200.vinet import VINet
    l, r = _pair(w, h, fmt, shift, seed=w + fmt)
    ref = V.flows(l, r, w, h, fmt, params).numpy()
    net = VINet(w, h, fmt, params=params, max_pairs=2)
    L = torch.from_numpy(np.stack([l, r])).cuda()
    R = torch.from_numpy(np.stack([r, l])).cuda()
    got = net.flows(L, R)
    torch.cuda.synchronize()
    g0 = got[0].cpu().numpy()
    err = np.abs(g0 - ref).max()
    scale = np.abs(ref).max()
    # bf16 operands through 30 layers: relative error of the residual flows
    assert err <= 0.03 * scale + 1e-3, (err, scale)
    # batch independence: pair 1 (swapped inputs) equals a single-pair run
    ref1 = V.flows(r, l, w, h, fmt, params).numpy()
    assert np.abs(got[1].cpu().numpy() - ref1).max() <= 0.03 * np.abs(ref1).max() + 1e-3


@pytest.mark.parametrize("w,h,fmt,shift", CASES)
def test_vinet_synth_on_oracle_flows(torch_cuda, params, w, h, fmt, shift):
    torch = torch_cuda
    from paper_2112_10603_b200.vinet import VINet
    l, r = _pair(w, h, fmt, shift, seed=w + fmt + 1)
    st = V.flows(l, r, w, h, fmt, params)
    st = st * 8.0  # exercise real displacements (several pixels) in the warp
    net = VINet(w, h, fmt, params=params, max_pairs=1)
    n = 5
    got = net.synth(torch.from_numpy(l[None]).cuda(), torch.from_numpy(r[None]).cuda(),
                    st[None].contiguous().cuda(), n)
    torch.cuda.synchronize()
    got = got[0].cpu().numpy()
    for j in range(1, n + 1):
        ref = V.synth(l, r, w, h, fmt, st, j / (n + 1))
        d = np.abs(got[j - 1].astype(int) - ref.astype(int))
        # identical fp32 formula; expf / division ulps can flip a rounding at .5
        assert d.max() <= 1 and (d > 0).mean() < 1e-3, (j, d.max(), (d > 0).mean())


def test_vinet_end_to_end_psnr(torch_cuda, params):
    torch = torch_cuda
    from paper_2112_10603_b200.vinet import VINet
    w, h, fmt = 448, 256, 2
    l, r = _pair(w, h, fmt, 3, seed=7)
    st = V.flows(l, r, w, h, fmt, params)
    net = VINet(w, h, fmt, params=params)
    got = net.dense_views(torch.from_numpy(l[None]).cuda(), torch.from_numpy(r[None]).cuda(), 3)[0].cpu().numpy()
    for j in range(1, 4):
        ref = V.synth(l, r, w, h, fmt, st, j / 4).astype(np.float64)
        mse = np.mean((got[j - 1].astype(np.float64) - ref) ** 2)
        psnr = 99.0 if mse == 0 else 10 * np.log10(255.0 ** 2 / mse)
        assert psnr >= 50.0, psnr


def test_vinet_rig_layout(torch_cuda, params):
    """fvv_vinet_rig = anchors + per-gap direct-t views in the fvv_rig_views layout."""
    torch = torch_cuda
    from paper_2112_10603_b200.vinet import VINet
    w, h, fmt, C, S = 192, 128, 1, 3, 2
    frames = [_pair(w, h, fmt, 2 * c, seed=30 + c)[0] for c in range(C)]
    cams = torch.from_numpy(np.stack(frames)).cuda()
    net = VINet(w, h, fmt, params=params, max_pairs=2)
    views = net.rig(cams, S)
    L, R = cams[:-1].contiguous(), cams[1:].contiguous()
    per_pair = net.dense_views(L, R, (1 << S) - 1)
    torch.cuda.synchronize()
    nv = (1 << S) - 1
    for c in range(C):
        assert torch.equal(views[c * (nv + 1)], cams[c])
    for c in range(C - 1):
        assert torch.equal(views[c * (nv + 1) + 1:c * (nv + 1) + 1 + nv], per_pair[c])


@pytest.mark.parametrize("w,h,fmt,C,S,vps", [(192, 128, 1, 4, 2, 4), (200, 128, 0, 3, 3, 5),
                                             (256, 192, 1, 5, 2, 1), (128, 64, 1, 3, 1, 2),
                                             (1920, 1080, 1, 3, 4, 16)])  # BASELINE 1080p geometry
def test_vinet_rig_clusters_fused_tiling(torch_cuda, params, w, h, fmt, C, S, vps):
    """fvv_vinet_rig_clusters (quarter tiles written by the synthesis epilogue) is
    byte-identical to fvv_vinet_rig + fvv_rig_clusters (server/pipeline.py:199-292)."""
    torch = torch_cuda
    from paper_2112_10603_b200.cluster import rig_clusters
    from paper_2112_10603_b200.vinet import VINet
    frames = [_pair(w, h, fmt, 2 * c + 1, seed=50 + c)[0] for c in range(C)]
    cams = torch.from_numpy(np.stack(frames)).cuda()
    net = VINet(w, h, fmt, params=params, max_pairs=2)  # C - 1 > 2 pairs: several chunks
    ref_views = net.rig(cams, S)
    ref_cl, ref_sizes = rig_clusters(ref_views, w, h, fmt, C, S, vps)
    views, cl, sizes = net.rig_clusters(cams, S, vps, out=torch.full_like(ref_cl, 77))
    torch.cuda.synchronize()
    assert sizes == ref_sizes
    assert torch.equal(views, ref_views)
    assert torch.equal(cl, ref_cl)


def test_vinet_flows_1080p_match_fp32_oracle(torch_cuda, params):
    """VINet at the BASELINE geometry (1920x1080 YUV420, canvas 1920x1088) vs the fp32
    oracle (run on the GPU with TF32 off, only to keep the checker fast)."""
    torch = torch_cuda
    from bench import synth_rig
    from paper_2112_10603_b200.vinet import VINet
    w, h, fmt = 1920, 1080, 1
    cams = synth_rig(w, h, fmt, 2, seed=1080)
    old = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
    torch.backends.cudnn.allow_tf32 = torch.backends.cuda.matmul.allow_tf32 = False
    try:
        ref = V.flows(cams[0], cams[1], w, h, fmt, params, device="cuda").numpy()
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = old
    net = VINet(w, h, fmt, params=params, max_pairs=1)
    got = net.flows(torch.from_numpy(cams[:1]).cuda(), torch.from_numpy(cams[1:]).cuda())[0].cpu().numpy()
    err = np.abs(got - ref)
    scale = np.abs(ref).max()
    assert err.max() <= 0.03 * scale + 1e-3, (err.max(), scale)
    # the 64-aligned canvas edge (rows 1024..1079, the last column tile) is no worse than the interior
    assert err[:, 1024:, :].max() <= 0.03 * scale + 1e-3
    assert float(np.mean(err)) <= 0.003 * scale + 1e-4
