"""RefineNet + ContextNet on B200 (refine.py) vs the fp32 torch oracle
(oracle/vinet_ref.py refine_view): bf16 convolutions through 21 layers, so
the bar is PSNR >= 50 dB on the refined uint8 views."""
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


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return 99.0 if mse == 0 else 10 * np.log10(255.0 ** 2 / mse)


@pytest.fixture(scope="module")
def params():
    from paper_2112_10603_b200.vinet_params import make_params, make_refine_params
    return make_params(0), make_refine_params(1)


@pytest.mark.parametrize("w,h,fmt", [(448, 256, 2), (256, 192, 1), (192, 128, 0), (200, 124, 1)])
def test_refined_views_match_fp32_oracle(torch_cuda, params, w, h, fmt):
    torch = torch_cuda
    from bench import synth_rig
    from paper_2112_10603_b200.refine import RefineNet
    vp, rp = params
    cams = synth_rig(w, h, fmt, 2, seed=w + fmt)
    st = V.flows(cams[0], cams[1], w, h, fmt, vp) * 4.0  # a few pixels of real displacement
    ref = RefineNet(w, h, fmt, params=rp, max_views=2)
    L = torch.from_numpy(cams[:1]).cuda()
    R = torch.from_numpy(cams[1:]).cuda()
    got = ref.views(L, R, st[None].cuda(), 3).cpu().numpy()  # 3 views in chunks of 2
    for j, t in enumerate((0.25, 0.5, 0.75)):
        want, _ = V.refine_view(cams[0], cams[1], w, h, fmt, st, t, rp)
        p = psnr(got[0, j], want)
        assert p >= 50.0, (j, p)


def test_refine_hook_on_the_sad_path(torch_cuda, params):
    """InterpConfig.refine = RefineNet.hook(): the reference's plugin seam
    (interp.py:144-145) refines the midpoint from the interpolation's mid
    flows and mask; equal (>= 50 dB) to the oracle fed the same diagnostics."""
    import torch
    import paper_2112_10603_b200 as fv
    from bench import synth_rig
    from oracle import oracle as O
    from paper_2112_10603_b200.refine import RefineNet
    _, rp = params
    w, h, fmt = 256, 192, 1
    cams = synth_rig(w, h, fmt, 2, seed=3)
    ref = RefineNet(w, h, fmt, params=rp)
    L, R = (fv.frame_from_packed(c, w, h, fmt) for c in cams)
    out = fv.interpolate(L, R, fv.InterpConfig(refine=ref.hook()))
    _, d = O.interpolate(cams[0], cams[1], w, h, fmt, with_diag=True)
    m = np.clip(d["mask"], 1e-12, 1 - 1e-12)
    st = torch.from_numpy(np.concatenate([np.moveaxis(d["flow_lr"] * -0.5, -1, 0),
                                          np.moveaxis(d["flow_rl"] * -0.5, -1, 0),
                                          np.log(m / (1 - m))[None]]).astype(np.float32))
    want, _ = V.refine_view(cams[0], cams[1], w, h, fmt, st, 0.5, rp)
    assert psnr(fv.packed(out), want) >= 50.0
