"""Parity of the CUDA path (through the C ABI) with the reference.

Bit-exact on every byte: uint8 output planes, f32 flows, f64 mask.  The
checker is the golden vectors the reference produced (tests/golden/) and
the CPU oracle (oracle/, itself pinned to those vectors by
tests/test_oracle_golden.py) on seeded inputs.
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FMT_NAMES = {0: "gray8", 1: "yuv420", 2: "rgb8"}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def _run_pairs(torch, w, h, fmt, lefts, rights, cfg=None):
    from paper_2112_10603_b200.interp import Interpolator
    eng = Interpolator(w, h, fmt, cfg, max_pairs=len(lefts))
    L = torch.from_numpy(np.stack(lefts)).cuda()
    R = torch.from_numpy(np.stack(rights)).cuda()
    out = eng.pairs(L, R)
    torch.cuda.synchronize()
    return eng, out.cpu().numpy()


@pytest.mark.parametrize("name", golden_names("interp"))
def test_interpolate_bit_exact_vs_golden(torch_cuda, name):
    g = load_golden(name)
    w, h, fmt = int(g["w"]), int(g["h"]), int(g["fmt"])
    eng, out = _run_pairs(torch_cuda, w, h, fmt, [g["left"]], [g["right"]])
    assert np.array_equal(out[0], g["out"]), f"{name}: {np.count_nonzero(out[0] != g['out'])} bytes differ"
    if "flow_lr" in g:
        flr, frl, m = eng.diagnostics(0)
        assert np.array_equal(flr.cpu().numpy(), g["flow_lr"])
        assert np.array_equal(frl.cpu().numpy(), g["flow_rl"])
        assert np.array_equal(m.cpu().numpy(), g["mask"])


def _rand_frames(rng, w, h, fmt, n):
    fb = O.frame_bytes(w, h, fmt)
    return [rng.integers(0, 256, fb, dtype=np.uint8) for _ in range(n)]


def _smooth_pair(rng, w, h, fmt, shift):
    """Smooth texture + its shifted copy (realistic flow), packed in `fmt`."""
    from scipy.ndimage import gaussian_filter
    big = gaussian_filter(rng.random((h + 8, w + 2 * abs(shift) + 8)) * 255.0, 3.0)
    big = (big - big.min()) / (np.ptp(big) + 1e-9) * 230 + 12
    a = big[4:4 + h, 4:4 + w]
    b = big[4:4 + h, 4 + shift:4 + shift + w]

    def pack(plane):
        p = np.rint(plane).astype(np.uint8)
        if fmt == 0:
            return p.reshape(-1)
        if fmt == 2:
            return np.stack([p, np.roll(p, 3, 1), 255 - p], -1).reshape(-1)
        c = p[::2, ::2]
        return np.concatenate([p.reshape(-1), c.reshape(-1), (255 - c).reshape(-1)])
    return pack(a), pack(b)


@pytest.mark.parametrize("w,h,fmt", [(64, 48, 0), (120, 68, 1), (100, 36, 2), (200, 140, 1),
                                     (36, 20, 0), (8, 8, 1), (4, 4, 0), (44, 12, 2),
                                     # 4:2:0 with W % 8 == 4 (a half last 8-column group, chroma width
                                     # % 4 == 2: the blend's unaligned chroma path)
                                     (132, 40, 1), (60, 28, 1), (52, 100, 0)])
def test_random_pairs_batched_vs_oracle(torch_cuda, w, h, fmt):
    rng = np.random.default_rng(w * 1000 + h * 10 + fmt)
    lefts, rights = [], []
    for i in range(3):
        a, b = _smooth_pair(rng, w, h, fmt, shift=i * 3 - 2)
        lefts.append(a)
        rights.append(b)
    ln, rn = _rand_frames(rng, w, h, fmt, 2)
    lefts.append(ln)
    rights.append(rn)
    _, out = _run_pairs(torch_cuda, w, h, fmt, lefts, rights)
    for i in range(len(lefts)):
        ref = O.interpolate(lefts[i], rights[i], w, h, fmt)
        assert np.array_equal(out[i], ref), f"pair {i}: {np.count_nonzero(out[i] != ref)} bytes differ"


@pytest.mark.parametrize("cfg", [dict(block_size=(4, 8, 2), search_radius=(6, 3, 1)),
                                 dict(block_size=(8, 4, 4), search_radius=(3, 2, 5)),
                                 dict(search_radius=(15, 6, 3), mask_epsilon=0.25)])
def test_nondefault_config_vs_oracle(torch_cuda, cfg):
    from paper_2112_10603_b200.interp import InterpConfig
    c = InterpConfig(**cfg)
    rng = np.random.default_rng(7)
    w, h, fmt = 96, 64, 1
    a, b = _smooth_pair(rng, w, h, fmt, 5)
    _, out = _run_pairs(torch_cuda, w, h, fmt, [a], [b], c)
    ref = O.interpolate(a, b, w, h, fmt, block_size=c.block_size, search_radius=c.search_radius,
                        eps=c.mask_epsilon)
    assert np.array_equal(out[0], ref)


def test_dense_views_vs_golden(torch_cuda):
    from paper_2112_10603_b200.interp import Interpolator
    g = load_golden("dense3_yuv420_64x48")
    eng = Interpolator(64, 48, 1, max_pairs=4)
    v = eng.dense(torch_cuda.from_numpy(g["left"]).cuda(), torch_cuda.from_numpy(g["right"]).cuda(), 3)
    assert np.array_equal(v.cpu().numpy(), g["out"])


def test_rig_views_and_clusters_vs_golden(torch_cuda):
    from paper_2112_10603_b200.interp import Interpolator
    from paper_2112_10603_b200.cluster import rig_clusters, downscale_device
    g = load_golden("rig3_s2_vps2_yuv420_64x48")
    w, h, fmt, stages, vps = 64, 48, 1, int(g["stages"]), int(g["vps"])
    cams = torch_cuda.from_numpy(g["cams"]).cuda()
    eng = Interpolator(w, h, fmt, max_pairs=2 * (1 << (stages - 1)))
    views = eng.rig(cams, stages)
    assert np.array_equal(views.cpu().numpy(), g["views"])
    q = downscale_device(views, w, h, fmt, 4)
    assert np.array_equal(q.cpu().numpy(), g["quarters"])
    out, sizes = rig_clusters(views, w, h, fmt, 3, stages, vps)
    assert list(sizes) == list(g["cluster_sizes"])
    assert np.array_equal(out.cpu().numpy(), g["clusters"])


def test_reference_api_roundtrip(torch_cuda):
    """interpolate()/dense_views() on host Frames, as the reference is called."""
    import paper_2112_10603_b200 as fv
    g = load_golden("scene_yuv420_96x72")
    L = fv.frame_from_packed(g["left"], 96, 72, 1)
    R = fv.frame_from_packed(g["right"], 96, 72, 1)
    out, diag = fv.interpolate(L, R, diagnostics=True)
    assert np.array_equal(fv.packed(out), g["out"])
    assert np.array_equal(diag.mask, g["mask"])
    assert diag.mask.min() >= 0.0 and diag.mask.max() <= 1.0
    views = fv.dense_views(L, R, 2)
    ref = O.dense_views(g["left"], g["right"], 96, 72, 1, 2)
    assert np.array_equal(np.stack([fv.packed(v) for v in views]), ref)
    seen = []
    cfg = fv.InterpConfig(refine=lambda f, d: (seen.append(d), f)[1])
    fv.interpolate(L, R, cfg)
    assert len(seen) == 1 and seen[0].mask is not None


def test_identity_and_errors(torch_cuda):
    import paper_2112_10603_b200 as fv
    rng = np.random.default_rng(3)
    img = fv.gray(rng.integers(0, 256, (48, 64), dtype=np.uint8))
    assert np.array_equal(fv.interpolate(img, img).planes[0], img.planes[0])
    with pytest.raises(ValueError):
        fv.interpolate(img, fv.gray(np.zeros((48, 60), np.uint8)))
    with pytest.raises(ValueError):
        fv.interpolate(fv.gray(np.zeros((30, 64), np.uint8)), fv.gray(np.zeros((30, 64), np.uint8)))
    with pytest.raises(ValueError):
        fv.dense_views(img, img, 0)
    with pytest.raises(ValueError):
        fv.dense_views(img, img, 7)


def test_full_1080p_pair_vs_oracle(torch_cuda):
    """BASELINE config size: one 1920x1080 YUV420 pair, bit-exact to the oracle."""
    rng = np.random.default_rng(1080)
    w, h, fmt = 1920, 1080, 1
    a, b = _smooth_pair(rng, w, h, fmt, 9)
    _, out = _run_pairs(torch_cuda, w, h, fmt, [a, b], [b, a])
    ref = O.interpolate(a, b, w, h, fmt)
    assert np.array_equal(out[0], ref), f"{np.count_nonzero(out[0] != ref)} bytes differ"
    ref2 = O.interpolate(b, a, w, h, fmt)
    assert np.array_equal(out[1], ref2)


@pytest.mark.parametrize("w,h,fmt,cams,stages,vps", [(40, 32, 1, 3, 2, 3), (96, 64, 0, 4, 3, 8),
                                                      (128, 72, 1, 2, 1, 1)])
def test_rig_clusters_vs_oracle(torch_cuda, w, h, fmt, cams, stages, vps):
    """Views and cluster frames of whole rigs (scalar and vector tiling paths)."""
    from paper_2112_10603_b200.interp import Interpolator
    from paper_2112_10603_b200.cluster import rig_clusters
    rng = np.random.default_rng(w + h + cams)
    frames = [_smooth_pair(rng, w, h, fmt, 4)[0] for _ in range(cams)]
    cams_np = np.stack(frames)
    eng = Interpolator(w, h, fmt, max_pairs=(cams - 1) * (1 << (stages - 1)))
    views = eng.rig(torch_cuda.from_numpy(cams_np).cuda(), stages)
    ref_views = O.rig_dense_views(cams_np, w, h, fmt, stages)
    assert np.array_equal(views.cpu().numpy(), ref_views)
    out, sizes = rig_clusters(views, w, h, fmt, cams, stages, vps)
    out = out.cpu().numpy()
    total = ref_views.shape[0]
    off = 0
    for c in range(cams):
        anchor = c << stages
        lo, hi = max(0, anchor - vps), min(total - 1, anchor + vps)
        smalls = np.stack([O.downscale(ref_views[i], w, h, fmt, 4) for i in range(lo, hi + 1) if i != anchor])
        ref, sw = O.assemble_cluster(ref_views[anchor], w, h, fmt, smalls)
        assert sizes[c] == ref.size
        assert np.array_equal(out[off:off + sizes[c]], ref), f"cluster {c}"
        off += sizes[c]


def test_rig_pipeline_device_resident_vs_golden(torch_cuda):
    """server/pipeline.py _interp + _stitch as one graph-captured device pipeline."""
    import paper_2112_10603_b200 as fv
    from paper_2112_10603_b200.pipeline import RigPipeline
    g = load_golden("rig3_s2_vps2_yuv420_64x48")
    w, h, stages, vps = 64, 48, int(g["stages"]), int(g["vps"])
    pipe = RigPipeline(w, h, 1, 3, stages, vps)
    cams = [fv.frame_from_packed(c, w, h, 1) for c in g["cams"]]
    for _ in range(2):  # replays of the captured graph give the same answer
        out = pipe.process_frames(cams)
        assert np.array_equal(pipe.views_host(), g["views"])
        got = np.concatenate([fv.packed(c.frame) for c in out])
        assert np.array_equal(got, g["clusters"])
    rects = np.array([[r.index, r.tier == "full", r.x, r.y, r.width, r.height]
                      for c in out for r in c.tile_map], np.int32)
    assert np.array_equal(rects, g["rects"])


@pytest.mark.parametrize("name", [n for n in golden_names("interp") if "lv0_flow_lr" in load_golden(n)])
def test_per_level_diagnostics_vs_golden(torch_cuda, name):
    """InterpDiagnostics.scales[s]: flows (f32) and match-error maps (f64), bitwise."""
    g = load_golden(name)
    w, h, fmt = int(g["w"]), int(g["h"]), int(g["fmt"])
    eng, _ = _run_pairs(torch_cuda, w, h, fmt, [g["left"]], [g["right"]])
    for s in range(3):
        flr, frl, elr, erl = (t.cpu().numpy() for t in eng.level_diagnostics(0, s))
        assert np.array_equal(flr, g[f"lv{s}_flow_lr"]), s
        assert np.array_equal(frl, g[f"lv{s}_flow_rl"]), s
        assert np.array_equal(elr, g[f"lv{s}_err_lr"]), s
        assert np.array_equal(erl, g[f"lv{s}_err_rl"]), s


@pytest.mark.parametrize("slots", [2, 3, 4])
def test_rig_pipeline_stream_ticks_overlapped(torch_cuda, slots):
    """Live-stream form (copies and consecutive ticks overlapped, one graph and
    compute stream per slot): every tick's clusters equal the golden ones.  More
    slots than two also checks that every slot's engine and views outlive
    their graph (allocations made after the capture must not reuse them)."""
    from paper_2112_10603_b200.pipeline import RigPipeline
    g = load_golden("rig3_s2_vps2_yuv420_64x48")
    pipe = RigPipeline(64, 48, 1, 3, int(g["stages"]), int(g["vps"]))
    cams = torch_cuda.from_numpy(g["cams"]).pin_memory()
    outs = [torch_cuda.empty(pipe.clusters.numel(), dtype=torch_cuda.uint8).pin_memory() for _ in range(7)]
    pipe.stream_ticks([cams] * 7, outs, slots=slots)
    torch_cuda.cuda.synchronize()
    junk = [torch_cuda.full((1 << 20,), 0x5A, dtype=torch_cuda.uint8, device="cuda") for _ in range(8)]
    outs2 = [torch_cuda.zeros_like(o).pin_memory() for o in outs]
    pipe.stream_ticks([cams] * 7, outs2, slots=slots)
    torch_cuda.cuda.synchronize()
    del junk
    for o in outs + outs2:
        assert np.array_equal(o.numpy(), g["clusters"])


def test_4k_pair_vs_oracle(torch_cuda):
    """BASELINE config 5 resolution (3840x2160 YUV420): one pair, bit-exact to the oracle."""
    rng = np.random.default_rng(2160)
    w, h, fmt = 3840, 2160, 1
    a, b = _smooth_pair(rng, w, h, fmt, 17)
    _, out = _run_pairs(torch_cuda, w, h, fmt, [a], [b])
    ref = O.interpolate(a, b, w, h, fmt)
    assert np.array_equal(out[0], ref), f"{np.count_nonzero(out[0] != ref)} bytes differ"


@pytest.mark.parametrize("name", [n for n in golden_names("interp") if "lv0_mask" in load_golden(n)])
def test_coarse_level_masks_vs_golden(torch_cuda, name):
    """ScaleDiagnostics.mask / blend_luma of levels 0-1 (interp.py:119-127), bitwise,
    through the engine and through interpolate(diagnostics=True)."""
    import paper_2112_10603_b200 as fv
    g = load_golden(name)
    w, h, fmt = int(g["w"]), int(g["h"]), int(g["fmt"])
    eng, _ = _run_pairs(torch_cuda, w, h, fmt, [g["left"]], [g["right"]])
    for s in range(2):
        m, b = (t.cpu().numpy() for t in eng.level_mask(0, s))
        assert np.array_equal(m, g[f"lv{s}_mask"]), s
        assert np.array_equal(b, g[f"lv{s}_blend"]), s
    _, diag = fv.interpolate(fv.frame_from_packed(g["left"], w, h, fmt), fv.frame_from_packed(g["right"], w, h, fmt),
                             diagnostics=True)
    assert np.array_equal(diag.scales[0].mask, g["lv0_mask"]) and np.array_equal(diag.scales[1].blend_luma,
                                                                                   g["lv1_blend"])
    assert diag.scales[2].blend_luma is None


def test_coarse_level_masks_1080p_vs_oracle(torch_cuda):
    """Levels 0-1 diagnostics at the BASELINE size vs the oracle fed the engine's
    (bitwise-verified) level flows."""
    from bench import synth_rig
    w, h, fmt = 1920, 1080, 1
    cams = synth_rig(w, h, fmt, 2, seed=11)
    eng, _ = _run_pairs(torch_cuda, w, h, fmt, [cams[0]], [cams[1]])
    pl, pr = O.luma_pyramid(cams[0], w, h, fmt), O.luma_pyramid(cams[1], w, h, fmt)
    for s in range(2):
        flr, frl, _, _ = (t.cpu().numpy() for t in eng.level_diagnostics(0, s))
        m_ref, b_ref = O.level_mask(pl[s], pr[s], flr, frl)
        m, b = (t.cpu().numpy() for t in eng.level_mask(0, s))
        assert np.array_equal(m, m_ref), s
        assert np.array_equal(b, b_ref), s
