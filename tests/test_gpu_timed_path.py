"""Parity of the code path the bench times, at the BASELINE sizes.

The headline number runs launch variants that small inputs never reach
(k_scan_carry's cooperative staging from ~600 one-warp CTAs, k_sadw's
stacked blocks from 2 CTAs per SM).  These tests run:

* the full cfg4 rig frame (8 cameras 1080p YUV420, 4 stages, 105 views, 8
  cluster frames) through `RigPipeline` -- the graph the bench replays --
  against the oracle, byte for byte (views and clusters);
* cfg2's `dense_views(..., 3)` at 1080p;
* every golden vector and ragged sizes with each launch variant FORCED on
  and off (fvv_engine_set_tuning), including partial scan chunks and plain launches
  instead of programmatic dependent launch;
* `assemble_cluster_frame` (k_assemble, the kernel plugin.install binds into
  the reference's `_stitch`) for gray and 4:2:0 with a part-empty last column;
* the drop-in `dense_views` from a 2-worker ThreadPoolExecutor, as the
  reference's `PipelineHandle._interp` calls it (server/pipeline.py:219-220,
  264-268).
"""
import numpy as np
import pytest

from bench import synth_rig
from conftest import golden_names, load_golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu

VARIANTS = {"all_on": dict(scan_coop_min=0, sadw_rb_min_ctas=0, mask_cols2=1, pdl=1),
            "all_off": dict(scan_coop_min=1 << 30, sadw_rb_min_ctas=1 << 30, mask_cols2=0, pdl=0)}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    return torch


def _pairs(torch, w, h, fmt, lefts, rights, cfg=None, **tuning):
    from paper_2112_10603_b200.interp import Interpolator
    eng = Interpolator(w, h, fmt, cfg, max_pairs=len(lefts)).set_tuning(**tuning)
    out = eng.pairs(torch.from_numpy(np.stack(lefts)).cuda(), torch.from_numpy(np.stack(rights)).cuda())
    torch.cuda.synchronize()
    return eng, out.cpu().numpy()


def test_cfg4_rig_frame_vs_oracle(torch_cuda):
    """The bench's timed step (BASELINE config 4), default launch variants: the
    56-pair stage runs k_scan_carry<COOP> (1904 CTAs) and stacked k_sadw."""
    from paper_2112_10603_b200.pipeline import RigPipeline
    import paper_2112_10603_b200 as fv
    W, H, fmt, C, stages, vps = 1920, 1080, 1, 8, 4, 16
    cams = synth_rig(W, H, fmt, C)
    pipe = RigPipeline(W, H, fmt, C, stages, vps)
    out = pipe.process_frames([fv.frame_from_packed(c, W, H, fmt) for c in cams])
    views = pipe.views_host()
    ref_views = O.rig_dense_views(cams, W, H, fmt, stages)
    bad = [i for i in range(ref_views.shape[0]) if not np.array_equal(views[i], ref_views[i])]
    assert not bad, f"views differing from the oracle: {bad}"
    total = ref_views.shape[0]
    for c, cf in enumerate(out):
        anchor = c << stages
        lo, hi = max(0, anchor - vps), min(total - 1, anchor + vps)
        smalls = np.stack([O.downscale(ref_views[i], W, H, fmt, 4) for i in range(lo, hi + 1) if i != anchor])
        ref, sw = O.assemble_cluster(ref_views[anchor], W, H, fmt, smalls)
        assert cf.frame.width == sw
        assert np.array_equal(fv.packed(cf.frame), ref), f"cluster {c}"


def test_cfg2_dense_1080p_vs_oracle(torch_cuda):
    """BASELINE config 2: one 1080p pair, dense_views(n=3) = 7 recursive views."""
    from paper_2112_10603_b200.interp import Interpolator
    cams = synth_rig(1920, 1080, 1, 2, seed=7)
    eng = Interpolator(1920, 1080, 1, max_pairs=4)
    v = eng.dense(torch_cuda.from_numpy(cams[0]).cuda(), torch_cuda.from_numpy(cams[1]).cuda(), 3)
    ref = O.dense_views(cams[0], cams[1], 1920, 1080, 1, 3)
    got = v.cpu().numpy()
    for i in range(7):
        assert np.array_equal(got[i], ref[i]), f"view {i + 1}: {np.count_nonzero(got[i] != ref[i])} bytes differ"


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("name", golden_names("interp"))
def test_goldens_with_forced_variants(torch_cuda, name, variant):
    g = load_golden(name)
    w, h, fmt = int(g["w"]), int(g["h"]), int(g["fmt"])
    eng, out = _pairs(torch_cuda, w, h, fmt, [g["left"]], [g["right"]], **VARIANTS[variant])
    assert np.array_equal(out[0], g["out"]), f"{name}/{variant}: {np.count_nonzero(out[0] != g['out'])} bytes differ"
    if "mask" in g:
        _, _, m = eng.diagnostics(0)
        assert np.array_equal(m.cpu().numpy(), g["mask"])


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("w,h,fmt", [(1000, 604, 1), (328, 200, 0), (264, 136, 2), (1920, 1080, 1)])
def test_ragged_batches_with_forced_variants(torch_cuda, w, h, fmt, variant):
    """Partial scan chunks (width % 64 != 0), ragged block grids, RGB: each
    launch variant forced, several pairs per launch, vs the oracle."""
    rng = np.random.default_rng(w * 7 + h + fmt)
    cams = synth_rig(w, h, fmt, 3, seed=int(rng.integers(1 << 30)))
    noise = rng.integers(0, 256, cams.shape[1], dtype=np.uint8)
    lefts, rights = [cams[0], cams[1], cams[2], noise], [cams[1], cams[2], cams[0], cams[0]]
    _, out = _pairs(torch_cuda, w, h, fmt, lefts, rights, **VARIANTS[variant])
    for i in range(len(lefts)):
        ref = O.interpolate(lefts[i], rights[i], w, h, fmt)
        assert np.array_equal(out[i], ref), f"pair {i}: {np.count_nonzero(out[i] != ref)} bytes differ"


def test_18_pair_1080p_batch_default_variants(torch_cuda):
    """>= 18 1080p pairs in ONE launch: 34 x 18 = 612 scan CTAs, so the default
    threshold (600) selects k_scan_carry<COOP> as in the timed cfg4 stages."""
    W, H, fmt = 1920, 1080, 1
    cams = synth_rig(W, H, fmt, 8, seed=18)
    lefts = [cams[i] for i in range(7)] + [cams[i + 1] for i in range(7)] + [cams[i] for i in range(4)]
    rights = [cams[i + 1] for i in range(7)] + [cams[i] for i in range(7)] + [cams[i + 2] for i in range(4)]
    _, out = _pairs(torch_cuda, W, H, fmt, lefts, rights)
    for i in range(len(lefts)):
        ref = O.interpolate(lefts[i], rights[i], W, H, fmt)
        assert np.array_equal(out[i], ref), f"pair {i}: {np.count_nonzero(out[i] != ref)} bytes differ"


@pytest.mark.parametrize("fmt,nsmall", [(0, 5), (1, 5), (1, 16), (0, 1), (1, 0)])
def test_assemble_cluster_frame_vs_oracle(torch_cuda, fmt, nsmall):
    """cluster.py:143-191 through k_assemble (what plugin.install binds into
    the reference's _stitch): anchor + quarter tiles, empty cells Y=0 / C=128."""
    import paper_2112_10603_b200 as fv
    from paper_2112_10603_b200.cluster import ClusterLayout, TileRef, assemble_cluster_frame
    W, H = 96, 64
    rng = np.random.default_rng(fmt * 100 + nsmall)
    anchor = rng.integers(0, 256, O.frame_bytes(W, H, fmt), dtype=np.uint8)
    smalls = [rng.integers(0, 256, O.frame_bytes(W // 4, H // 4, fmt), dtype=np.uint8) for _ in range(nsmall)]
    tiles = [TileRef(i, "quarter") for i in range(nsmall // 2)] + [TileRef(nsmall // 2, "full")] + \
            [TileRef(i + 1, "quarter") for i in range(nsmall // 2, nsmall)]
    lay = ClusterLayout(3, nsmall // 2, 0, nsmall, 8, tuple(tiles))
    cf = assemble_cluster_frame(fv.frame_from_packed(anchor, W, H, fmt),
                                [fv.frame_from_packed(s, W // 4, H // 4, fmt) for s in smalls], lay)
    ref, sw = O.assemble_cluster(anchor, W, H, fmt, np.stack(smalls) if smalls else np.zeros((0, 0), np.uint8))
    assert cf.frame.width == sw and cf.cluster_id == 3
    assert np.array_equal(fv.packed(cf.frame), ref)
    full = [r for r in cf.tile_map if r.tier == "full"]
    assert len(full) == 1 and (full[0].x, full[0].y, full[0].width, full[0].height) == (0, 0, W, H)
    quarter = [r for r in cf.tile_map if r.tier == "quarter"]
    for i, r in enumerate(quarter):
        assert (r.x, r.y) == (W + (i // 4) * (W // 4), (i % 4) * (H // 4))
        assert np.array_equal(fv.packed(cf.crop(r)), smalls[i])


def test_drop_in_dense_views_from_two_threads(torch_cuda):
    """20 concurrent dense_views calls on distinct pairs from a 2-worker pool
    (the reference's PipelineHandle._interp pattern): every result bitwise."""
    from concurrent.futures import ThreadPoolExecutor
    import paper_2112_10603_b200 as fv
    W, H, fmt = 160, 96, 1
    cams = synth_rig(W, H, fmt, 21, seed=5)
    frames = [fv.frame_from_packed(c, W, H, fmt) for c in cams]

    def job(i):
        views = fv.dense_views(frames[i], frames[i + 1], 2)
        return np.stack([fv.packed(v) for v in views])

    with ThreadPoolExecutor(max_workers=2) as ex:
        got = list(ex.map(job, range(20)))
    for i in range(20):
        ref = O.dense_views(cams[i], cams[i + 1], W, H, fmt, 2)
        assert np.array_equal(got[i], ref), f"gap {i}"
    # interpolate() with diagnostics from two threads as well
    with ThreadPoolExecutor(max_workers=2) as ex:
        res = list(ex.map(lambda i: fv.interpolate(frames[i], frames[i + 1], diagnostics=True), range(8)))
    for i, (f, d) in enumerate(res):
        ref, diag = O.interpolate(cams[i], cams[i + 1], W, H, fmt, with_diag=True)
        assert np.array_equal(fv.packed(f), ref)
        assert np.array_equal(d.mask, diag["mask"])


@pytest.mark.parametrize("world,W,H,C,stages,vps", [(2, 1920, 1080, 8, 4, 16), (3, 96, 64, 5, 2, 3),
                                                     (8, 64, 48, 8, 2, 4)])
def test_gap_sharded_rig_device_vs_unsharded(torch_cuda, world, W, H, C, stages, vps):
    """Every rank's share of a gap-sharded rig frame (GapShardedRig), run one
    rank after another on this GPU with the halo handed over by a device copy
    (the NCCL exchange itself is covered on gloo): the gathered clusters equal
    fvv_rig_clusters of the whole rig, byte for byte."""
    import torch
    from paper_2112_10603_b200.cluster import rig_clusters
    from paper_2112_10603_b200.interp import Interpolator
    from paper_2112_10603_b200.shard import GapShardedRig
    fmt = 1
    cams = torch.from_numpy(synth_rig(W, H, fmt, C, seed=3)).cuda()
    ranks = [GapShardedRig(W, H, fmt, C, stages, vps, r, world) for r in range(world)]
    for rk in ranks:
        p = rk.plan
        if p.active:
            rk.cams[:len(p.cams)].copy_(cams[p.cams.start:p.cams.stop])
        rk.compute()
    for rk in ranks:
        if rk.plan.halo_in is not None:
            rk.halo_recv.copy_(ranks[rk.plan.halo_in[0]].halo_send)
        rk.stitch()
    torch.cuda.synchronize()
    got = torch.cat([rk.clusters[:sum(rk.cluster_sizes)] for rk in ranks if rk.cluster_sizes]).cpu().numpy()
    eng = Interpolator(W, H, fmt, max_pairs=(C - 1) << (stages - 1))
    views = eng.rig(cams, stages)
    ref, sizes = rig_clusters(views, W, H, fmt, C, stages, vps)
    assert got.size == sum(sizes)
    assert np.array_equal(got, ref.cpu().numpy())


def _sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_1080p_pair_vs_reference_golden(torch_cuda):
    """The CUDA path against the REFERENCE's own 1080p output (no oracle in
    between): tests/golden/ref1080_pair.npz, inputs regenerated from the seed."""
    g = load_golden("ref1080_pair")
    w, h = int(g["w"]), int(g["h"])
    cams = synth_rig(w, h, 1, int(g["cams"]), seed=int(g["seed"]))
    eng, out = _pairs(torch_cuda, w, h, 1, [cams[0]], [cams[1]])
    assert np.array_equal(out[0], g["out"])
    flr, frl, m = (t.cpu().numpy() for t in eng.diagnostics(0))
    assert _sha(flr) == str(g["flow_lr_sha"]) and _sha(frl) == str(g["flow_rl_sha"])
    assert _sha(m) == str(g["mask_sha"])


def test_cfg3_rig_vs_reference_golden(torch_cuda):
    """BASELINE config 3 through RigPipeline (graph replay): all 45 views' and 4
    cluster frames' SHA-256 equal the reference's (tests/golden/ref1080_cfg3.npz),
    and the tile maps equal the reference's TileRects."""
    import paper_2112_10603_b200 as fv
    from paper_2112_10603_b200.pipeline import RigPipeline
    g = load_golden("ref1080_cfg3")
    w, h, C, S, vps = int(g["w"]), int(g["h"]), int(g["cams"]), int(g["stages"]), int(g["vps"])
    cams = synth_rig(w, h, 1, C, seed=int(g["seed"]))
    pipe = RigPipeline(w, h, 1, C, S, vps)
    out = pipe.process_frames([fv.frame_from_packed(c, w, h, 1) for c in cams])
    views = pipe.views_host()
    assert [_sha(v) for v in views] == [str(s) for s in g["view_sha"]]
    assert [_sha(fv.packed(c.frame)) for c in out] == [str(s) for s in g["cluster_sha"]]
    rects = np.array([[r.index, r.tier == "full", r.x, r.y, r.width, r.height] for c in out for r in c.tile_map],
                     np.int32)
    assert np.array_equal(rects, g["rects"])


def test_device_rig_stages_two_threads_vs_golden(torch_cuda):
    """pipeline.DeviceRigStages as plugin.install(fvv, pipeline=True) drives it:
    _interp and _stitch on their own threads joined by a bounded queue (the
    reference's channel back-pressure), 8 ticks cycling 3 device slots; every
    tick's cluster frames, tile maps and views equal the reference's golden."""
    import queue
    import threading
    import paper_2112_10603_b200 as fv
    from paper_2112_10603_b200.pipeline import DeviceRigStages
    g = load_golden("rig3_s2_vps2_yuv420_64x48")
    w, h, stages, vps = 64, 48, int(g["stages"]), int(g["vps"])
    st = DeviceRigStages(w, h, 1, 3, stages, vps, slots=3)
    cams = [fv.frame_from_packed(c, w, h, 1) for c in g["cams"]]
    q, results, errors = queue.Queue(maxsize=1), [], []

    def interp_worker():
        try:
            for t in range(8):
                q.put(st.interp([c.with_timestamp(t) for c in cams]))
            q.put(None)
        except BaseException as e:  # noqa: BLE001
            errors.append(e)
            q.put(None)

    def stitch_worker():
        try:
            while (slot := q.get()) is not None:
                results.append((slot, st.stitch(slot)))
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=interp_worker), threading.Thread(target=stitch_worker)]
    for t in th:
        t.start()
    for t in th:
        t.join(120)
    assert not errors, errors
    assert len(results) == 8
    for t, (slot, out) in enumerate(results):
        assert np.array_equal(np.concatenate([fv.packed(c.frame) for c in out]), g["clusters"]), f"tick {t}"
        assert all(c.frame.timestamp == t for c in out)
        rects = np.array([[r.index, r.tier == "full", r.x, r.y, r.width, r.height] for c in out for r in c.tile_map],
                         np.int32)
        assert np.array_equal(rects, g["rects"])
    assert np.array_equal(st.views_host(results[-1][0]), g["views"])


@pytest.mark.parametrize("w,h,fmt,stages", [(256, 192, 1, 3), (192, 128, 0, 2), (200, 124, 2, 4)])
def test_direct_t_dense_views(torch_cuda, w, h, fmt, stages):
    """dense_views mode "direct" (fvv_dense_views FVV_DENSE_DIRECT): the t = 1/2 view
    is the reference's midpoint bit for bit; every other view equals the direct-t
    synthesis of the oracle's flows and mask (vinet_ref.synth, fp32) within 1 level."""
    import torch
    from oracle import vinet_ref as V
    from paper_2112_10603_b200.interp import Interpolator
    cams = synth_rig(w, h, fmt, 2, seed=w + stages)
    eng = Interpolator(w, h, fmt, max_pairs=1)
    got = eng.dense(torch.from_numpy(cams[0]).cuda(), torch.from_numpy(cams[1]).cuda(), stages, mode=1).cpu().numpy()
    nv = (1 << stages) - 1
    mid, d = O.interpolate(cams[0], cams[1], w, h, fmt, with_diag=True)
    assert np.array_equal(got[nv // 2], mid)
    m = np.clip(d["mask"], 1e-7, 1 - 1e-7)
    st = torch.from_numpy(np.concatenate([np.moveaxis(d["flow_lr"] * np.float32(-0.5), -1, 0),
                                          np.moveaxis(d["flow_rl"] * np.float32(-0.5), -1, 0),
                                          np.log(m / (1 - m))[None]]).astype(np.float32))
    for j in range(nv):
        if j == nv // 2:
            continue
        want = V.synth(cams[0], cams[1], w, h, fmt, st, (j + 1) / (nv + 1))
        diff = np.abs(got[j].astype(int) - want.astype(int))
        assert diff.max() <= 1 and np.mean(diff) < 0.01, (j, diff.max(), np.mean(diff))


def test_dense_views_modes_through_the_reference_api(torch_cuda):
    """dense_views(..., mode=) on host Frames: recursive (bit-exact vs the oracle),
    direct (midpoint bit-exact) and vinet (the CNN path)."""
    import paper_2112_10603_b200 as fv
    w, h, fmt = 128, 96, 1
    cams = synth_rig(w, h, fmt, 2, seed=9)
    L, R = (fv.frame_from_packed(c, w, h, fmt) for c in cams)
    rec = np.stack([fv.packed(v) for v in fv.dense_views(L, R, 2)])
    assert np.array_equal(rec, O.dense_views(cams[0], cams[1], w, h, fmt, 2))
    dir_ = np.stack([fv.packed(v) for v in fv.dense_views(L, R, 2, mode="direct")])
    assert np.array_equal(dir_[1], rec[1])
    vin = fv.dense_views(L, R, 2, mode="vinet")
    assert len(vin) == 3 and vin[0].width == w
    with pytest.raises(ValueError):
        fv.dense_views(L, R, 2, mode="nope")


@pytest.mark.parametrize("w,h,fmt,C,stages", [(200, 124, 1, 4, 3), (1920, 1080, 1, 3, 4)])
def test_direct_t_rig_equals_per_gap_direct_dense(torch_cuda, w, h, fmt, C, stages):
    """fvv_rig_views_mode(DIRECT): all gaps in one launch == fvv_dense_views(DIRECT)
    gap by gap (anchors, bit-exact midpoints, synthesized views), byte for byte."""
    import torch
    from paper_2112_10603_b200.interp import Interpolator
    cams = torch.from_numpy(synth_rig(w, h, fmt, C, seed=C + stages)).cuda()
    eng = Interpolator(w, h, fmt, max_pairs=C - 1)
    views = eng.rig(cams, stages, mode=1).cpu().numpy()
    one = Interpolator(w, h, fmt, max_pairs=1)
    step = 1 << stages
    for c in range(C - 1):
        d = one.dense(cams[c], cams[c + 1], stages, mode=1).cpu().numpy()
        assert np.array_equal(views[c * step + 1:(c + 1) * step], d), c
        assert np.array_equal(views[c * step], cams[c].cpu().numpy())
    assert np.array_equal(views[-1], cams[-1].cpu().numpy())


@pytest.mark.parametrize("cfg,w,h,fmt", [
    (dict(block_size=(6, 5, 3)), 96, 72, 1),
    (dict(block_size=(8, 8, 6), search_radius=(12, 4, 3)), 120, 68, 0),
    (dict(block_size=(3, 3, 3), search_radius=(4, 2, 1), mask_epsilon=0.05), 64, 48, 2),
    (dict(search_radius=(30, 4, 2)), 128, 96, 1),      # max_span 130 > 120
    (dict(block_size=(7, 9, 5)), 1920, 1080, 1),       # the literal path at the BASELINE size
])
def test_literal_path_for_any_config_vs_oracle(torch_cuda, cfg, w, h, fmt):
    """InterpConfig values outside the fixed-point domain (interp.py:32-36 accepts any
    block >= 2, radius >= 1): the literal path, bit-exact vs the oracle -- output
    planes, final flows and mask, per-level flows / errors / coarse masks."""
    import paper_2112_10603_b200 as fv
    c = fv.InterpConfig(**cfg)
    cams = synth_rig(w, h, fmt, 3, seed=w + fmt)
    lefts, rights = [cams[0], cams[1]], [cams[1], cams[2]]
    eng, out = _pairs(torch_cuda, w, h, fmt, lefts, rights, c)
    kw = dict(block_size=c.block_size, search_radius=c.search_radius, eps=c.mask_epsilon)
    for i in range(2):
        ref = O.interpolate(lefts[i], rights[i], w, h, fmt, **kw)
        assert np.array_equal(out[i], ref), f"pair {i}: {np.count_nonzero(out[i] != ref)} bytes differ"
    ref, d = O.interpolate(lefts[1], rights[1], w, h, fmt, with_diag=True, **kw)
    flr, frl, m = (t.cpu().numpy() for t in eng.diagnostics(1))
    assert np.array_equal(flr, d["flow_lr"]) and np.array_equal(frl, d["flow_rl"]) and np.array_equal(m, d["mask"])
    if w <= 128:  # reference-API route incl. per-level diagnostics
        L, R = (fv.frame_from_packed(x, w, h, fmt) for x in (lefts[1], rights[1]))
        res, diag = fv.interpolate(L, R, c, diagnostics=True)
        assert np.array_equal(fv.packed(res), ref)
        pl, pr = O.luma_pyramid(lefts[1], w, h, fmt), O.luma_pyramid(rights[1], w, h, fmt)
        prev = None
        for s in range(3):
            (fl, fr), _, (el, er) = O.estimate_flow_level(pl[s], pr[s], prev, c.search_radius[s], c.block_size[s])
            sd = diag.scales[s]
            assert np.array_equal(sd.flow_lr.vectors, fl) and np.array_equal(sd.flow_rl.vectors, fr), s
            assert np.array_equal(sd.match_error_lr, el) and np.array_equal(sd.match_error_rl, er), s
            if s < 2:
                mm, bb = O.level_mask(pl[s], pr[s], fl, fr, c.mask_epsilon)
                assert np.array_equal(sd.mask, mm) and np.array_equal(sd.blend_luma, bb), s
            prev = (fl, fr)
