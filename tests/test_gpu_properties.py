"""The reference's property tests of the flow/interp path, run on the CUDA path.

Each test restates one known-answer or threshold test of the reference suite
(cited per test) on synthetic textures generated here, through the public
mirror API (`paper_2112_10603_b200.interpolate(..., diagnostics=True)`), so
the per-level flows and match errors come from the C-ABI diagnostics entry
points (`fvv_interp_level_diagnostics`, `fvv_interp_diagnostics`).  The
byte-level parity itself is in test_gpu_parity.py; these check that the
properties the reference asserts hold on the device path at sizes larger
than the golden fixtures.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fv():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2112_10603_b200 as fv
    return fv


def _texture(seed, h, w, sigma=1.6):
    """Band-limited noise in 28..218 (the reference's value-noise range)."""
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(seed)
    t = gaussian_filter(rng.random((h, w)), sigma)
    t = (t - t.min()) / (np.ptp(t) + 1e-12)
    return np.rint(28 + 190 * t).astype(np.uint8)


def _shifted_pair(fv, seed, h, w, shift):
    """L(u) == R(u + shift) exactly for an integer shift (test_flow_warp.py:25-34)."""
    tex = _texture(seed, h, w + abs(shift))
    if shift >= 0:
        left, right = tex[:, shift:shift + w], tex[:, :w]
    else:
        left, right = tex[:, :w], tex[:, -shift:-shift + w]
    return fv.gray(left.copy()), fv.gray(right.copy())


def _up2(v, w_out, h_out):
    """upscale_flow (flow.py:47-54 -> _kernels.py:136-167): sample at
    (i + 0.5) * (n_in / n_out) - 0.5, clamp, x-lerp then y-lerp, times 2."""
    h_in, w_in = v.shape[:2]
    sy = np.clip((np.arange(h_out) + 0.5) * (h_in / h_out) - 0.5, 0, h_in - 1)
    sx = np.clip((np.arange(w_out) + 0.5) * (w_in / w_out) - 0.5, 0, w_in - 1)
    y0 = np.minimum(np.floor(sy).astype(int), max(h_in - 2, 0))
    x0 = np.minimum(np.floor(sx).astype(int), max(w_in - 2, 0))
    y1, x1 = np.minimum(y0 + 1, h_in - 1), np.minimum(x0 + 1, w_in - 1)
    fy, fx = (sy - y0)[:, None, None], (sx - x0)[None, :, None]
    a = v.astype(np.float64)
    top = (1 - fx) * a[y0][:, x0] + fx * a[y0][:, x1]
    bot = (1 - fx) * a[y1][:, x0] + fx * a[y1][:, x1]
    return ((1 - fy) * top + fy * bot) * 2.0


def test_identical_inputs_zero_flow(fv):
    """test_flow_warp.py:80-85 and test_interp.py:14-21: zero flow, zero error, I -> I."""
    img = fv.gray(_texture(5, 96, 128))
    out, diag = fv.interpolate(img, img, diagnostics=True)
    assert np.array_equal(out.planes[0], img.planes[0])
    for s in diag.scales:
        assert s.flow_lr.max_magnitude() == 0.0 and s.flow_rl.max_magnitude() == 0.0
        assert s.match_error_lr.max() == 0.0 and s.match_error_rl.max() == 0.0


@pytest.mark.parametrize("shift", [6, -6, 17])
def test_flow_recovers_global_shift(fv, shift):
    """test_flow_warp.py:88-93: the median finest-level flow is the shift within 0.5 px."""
    left, right = _shifted_pair(fv, 7, 96, 160, shift)
    _, diag = fv.interpolate(left, right, diagnostics=True)
    flr = diag.scales[-1].flow_lr.vectors
    frl = diag.scales[-1].flow_rl.vectors
    assert abs(np.median(flr[..., 0]) - shift) <= 0.5
    assert abs(np.median(flr[..., 1])) <= 0.5
    assert abs(np.median(frl[..., 0]) + shift) <= 0.5


def test_flow_saturates_beyond_span(fv):
    """test_flow_warp.py:96-105: |flow| <= max_span = 58, and the failed match shows in the error."""
    cfg = fv.InterpConfig()
    assert cfg.max_span == 58
    left, right = _shifted_pair(fv, 3, 96, 160, 100)
    good_l, good_r = _shifted_pair(fv, 3, 96, 160, 4)
    _, diag = fv.interpolate(left, right, diagnostics=True)
    _, diag_good = fv.interpolate(good_l, good_r, diagnostics=True)
    worst = diag.scales[-1]
    assert np.abs(worst.flow_lr.vectors).max() <= cfg.max_span
    assert worst.match_error_lr.mean() > 4 * diag_good.scales[-1].match_error_lr.mean()


def test_flow_residual_bounded_by_radius(fv):
    """test_flow_warp.py:108-117: each level's flow differs from the upscaled coarser flow by
    at most that level's search radius."""
    cfg = fv.InterpConfig()
    a = _texture(11, 120, 192, sigma=2.5)
    yy, xx = np.mgrid[0:120, 0:192]
    # a smooth non-uniform disparity field (3..9 px) so every level has a residual to find
    disp = 3 + 6 * (xx / 191.0) * (0.5 + 0.5 * np.sin(yy / 19.0))
    src_x = np.clip(xx + disp, 0, 191)
    x0 = np.floor(src_x).astype(int)
    x1 = np.minimum(x0 + 1, 191)
    f = src_x - x0
    b = np.rint((1 - f) * a[yy, x0] + f * a[yy, x1]).astype(np.uint8)
    _, diag = fv.interpolate(fv.gray(b), fv.gray(a), cfg, diagnostics=True)
    for s in (1, 2):
        for name in ("flow_lr", "flow_rl"):
            prev = getattr(diag.scales[s - 1], name).vectors
            cur = getattr(diag.scales[s], name).vectors
            up = _up2(prev, cur.shape[1], cur.shape[0])
            assert np.abs(cur - up).max() <= cfg.search_radius[s] + 1e-4, (s, name)


def test_mirror_symmetry(fv):
    """test_interp.py:35-47: interpolating the mirrored pair mirrors the result (>= 99 % within 1)."""
    left, right = _shifted_pair(fv, 21, 96, 160, 5)

    def mirror(fr):
        return fv.frame_from_planes([np.ascontiguousarray(p[:, ::-1]) for p in fr.planes], fr.format,
                                    fr.timestamp)

    a = fv.interpolate(left, right)
    b = mirror(fv.interpolate(mirror(right), mirror(left)))
    d = np.abs(a.planes[0].astype(int) - b.planes[0].astype(int))
    assert np.mean(d <= 1) >= 0.99


def test_mask_within_bounds_and_flow_mid(fv):
    """test_interp.py:50-55 (mask in [0, 1]) and interp.py:131-132 (mid flows = -0.5 x flow)."""
    left, right = _shifted_pair(fv, 9, 96, 160, 8)
    _, diag = fv.interpolate(left, right, diagnostics=True)
    assert diag.mask.min() >= 0.0 and diag.mask.max() <= 1.0
    assert diag.mask.dtype == np.float64
    assert np.array_equal(diag.flow_mid_left.vectors,
                          diag.scales[-1].flow_lr.vectors * np.float32(-0.5))
