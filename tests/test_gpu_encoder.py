"""The FVT1 encoder hand-off on B200 (encoder.RigEncoder) vs records the
reference's own encoder stage wrote (server/pipeline.py:294-318,
codec.TileEncoder; tests/golden/make_golden_encoder.py): byte-identical I and
P records for the lossy DCT path (q75, gop 2) and the lossless lifting path
(q100, gop 3), with the reconstruction carried on the device between ticks."""
import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("setting,quality,gop", [("q75", 75, 2), ("q100", 100, 3)])
def test_rig_encoder_records_equal_reference(setting, quality, gop):
    import torch
    from paper_2112_10603_b200.cluster import build_layouts
    from paper_2112_10603_b200.encoder import RigEncoder
    from paper_2112_10603_b200.viewmodel import ViewIndexModel
    g = load_golden("encoder_rig3_yuv420_64x48")
    W, H, C, S, vps, T = (int(g[k]) for k in ("w", "h", "cams", "stages", "vps", "ticks"))
    enc = RigEncoder(build_layouts(ViewIndexModel(C, S), vps), W, H, 1, quality=quality, gop=gop)
    lens = g[f"{setting}_lengths"]
    blob = g[f"{setting}_records"].tobytes()
    offs = np.concatenate([[0], np.cumsum(lens)])
    want = [blob[offs[i]:offs[i + 1]] for i in range(len(lens))]
    got = []
    for t in range(T):
        recs = enc.encode(torch.from_numpy(g["clusters"][t]).cuda())
        got += [r for c in recs for r in c]
    assert len(got) == len(want)
    bad = [i for i, (a, b) in enumerate(zip(got, want)) if a != b]
    assert not bad, f"records differing: {bad[:10]} of {len(want)}"


def test_device_rig_stages_encode_hand_off():
    """DeviceRigStages.stitch_device + .encode (the plugin's _stitch/_encode
    hooks): records of 3 ticks equal a RigEncoder fed the golden cluster frames."""
    import torch
    import paper_2112_10603_b200 as fv
    from paper_2112_10603_b200.cluster import build_layouts
    from paper_2112_10603_b200.encoder import RigEncoder
    from paper_2112_10603_b200.pipeline import DeviceRigStages
    from paper_2112_10603_b200.viewmodel import ViewIndexModel
    g = load_golden("rig3_s2_vps2_yuv420_64x48")
    w, h, S, vps = 64, 48, int(g["stages"]), int(g["vps"])
    st = DeviceRigStages(w, h, 1, 3, S, vps, slots=3)
    cams = [fv.frame_from_packed(c, w, h, 1) for c in g["cams"]]
    ref = RigEncoder(build_layouts(ViewIndexModel(3, S), vps), w, h, 1, quality=60, gop=2)
    for t in range(3):
        slot = st.interp(cams)
        st.stitch_device(slot)
        got = st.encode(slot, 60, 2)
        assert np.array_equal(st.clusters[slot].cpu().numpy(), g["clusters"])
        want = ref.encode(torch.from_numpy(g["clusters"]).cuda())
        assert got == want, t
