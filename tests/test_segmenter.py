"""TS/HLS packaging (segmenter.py, csrc/ts_mux.cpp) -- host code, CPU tests.

Byte-identical to the reference's mpegts.mux_segment on golden segments
(tests/golden/make_golden_ts.py) and, where /root/reference exists, on random
segments and the reference's playlist rendering; the pipeline's per-cluster
concurrent muxing gives the same bytes as one-by-one."""
import numpy as np
import pytest

import refimpl
from conftest import load_golden


def _cases(seed):
    """The golden generator's records (tests/golden/make_golden_ts.py), same seed."""
    from golden.make_golden_ts import records
    rng = np.random.default_rng(seed)
    return {"tiny": records(rng, 3, 2, 5, 20), "multi": records(rng, 6, 5, 100, 2000),
            "big": records(rng, 2, 3, 30000, 40000)}


def _frames(g, name):
    return _cases(int(g["seed"]))[name]


@pytest.mark.parametrize("name", ["tiny", "multi", "big"])
def test_segments_equal_reference_goldens(name):
    from paper_2112_10603_b200.segmenter import mux_segment
    g = load_golden("ts_segments")
    import hashlib
    got = mux_segment(_frames(g, name), int(g[f"{name}_fps"]), int(g[f"{name}_start"]))
    assert len(got) == int(g[f"{name}_size"])
    if f"{name}_segment" in g:
        assert got == g[f"{name}_segment"].tobytes()
    assert hashlib.sha256(got).hexdigest() == str(g[f"{name}_sha256"])


def test_concurrent_cluster_muxing_and_gop_check():
    from paper_2112_10603_b200.segmenter import GopAlignmentError, SegmentMuxer, mux_segment
    g = load_golden("ts_segments")
    per = [_frames(g, n) for n in ("tiny", "multi", "big")]
    m = SegmentMuxer(threads=3)
    got = m.mux_clusters(per, 30, 900)
    assert got == [mux_segment(f, 30, 900) for f in per]
    bad = [[b"\x01abc", b"\x00x"]]
    with pytest.raises(GopAlignmentError):
        mux_segment(bad, 30)
    with pytest.raises(ValueError):
        mux_segment(bad, 0)


@pytest.mark.reference
@pytest.mark.skipif(not refimpl.available(), reason="/root/reference not present")
def test_random_segments_and_playlists_equal_reference():
    refimpl.load()
    from fvv import mpegts, playlist
    from paper_2112_10603_b200.segmenter import PlaylistWindow, mux_segment
    rng = np.random.default_rng(7)
    for trial in range(20):
        nf, nt = int(rng.integers(1, 6)), int(rng.integers(1, 9))
        frames = [[bytes([0 if f == 0 else 1]) + rng.integers(0, 256, int(rng.integers(0, 3000)),
                                                              dtype=np.uint8).tobytes() for _ in range(nt)]
                  for f in range(nf)]
        fps, start = int(rng.choice([24, 25, 30, 60, 7])), int(rng.integers(0, 1 << 33))
        assert mux_segment(frames, fps, start) == mpegts.mux_segment(frames, fps, start), trial
    ref = playlist.new_playlist(2.0, 3)
    ours = PlaylistWindow.for_segments(2.0, 3)
    for seq in range(7):
        ref, text = playlist.rotate_playlist(ref, seq, 2.0 + 0.001 * seq)
        assert ours.rotate(seq, 2.0 + 0.001 * seq) == text
    assert ours.end() == playlist.end_playlist(ref)[1]
