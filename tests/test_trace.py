"""EDGT trace I/O and the device analyze-trace pass.

Mirrors the reference's TestTraceRoundTrip (pkg/tests/test_grad_source.py:25-72)
and TestAnalyzeTrace (pkg/tests/test_cli.py:250-325); the analyze outputs are
checked against tests/golden/trace.json, written by the reference's own
``analyze-trace`` (tests/golden/make_trace_golden.py).
"""

import csv
import hashlib
import io

import numpy as np
import pytest

from paper_2511_10333_b200.errors import TraceFormatError
from paper_2511_10333_b200.trace import analyze_trace, read_trace_header, replay_trace, write_trace
from tests.golden.specs import TRACE_SPEC, trace_frames
from tests.helpers import load_json

GOLD = load_json("trace.json")


def _rows(text):
    rows = list(csv.reader(io.StringIO(text)))
    return rows[0], rows[1:]


# ---- host-side format (no GPU)

def test_writer_bytes_match_reference(tmp_path):
    path = tmp_path / "t.edgt"
    assert write_trace(path, trace_frames()) == TRACE_SPEC["iterations"]
    assert hashlib.sha256(path.read_bytes()).hexdigest() == GOLD["trace_sha256"]
    count, shapes = read_trace_header(path)
    assert count == TRACE_SPEC["iterations"]
    assert shapes == [tuple(s) for s in TRACE_SPEC["shapes"]]


def test_empty_trace(tmp_path):
    path = tmp_path / "empty.edgt"
    assert write_trace(path, []) == 0
    assert read_trace_header(path) == (0, [])
    assert list(replay_trace(path)) == []


def test_bad_magic(tmp_path):
    path = tmp_path / "bad.edgt"
    path.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(TraceFormatError, match="magic"):
        list(replay_trace(path))


def test_bad_version_and_width(tmp_path):
    import struct
    p = tmp_path / "v.edgt"
    p.write_bytes(struct.pack("<4sHHIH", b"EDGT", 2, 0, 0, 4))
    with pytest.raises(TraceFormatError, match="version"):
        read_trace_header(p)
    p.write_bytes(struct.pack("<4sHHIH", b"EDGT", 1, 0, 0, 8))
    with pytest.raises(TraceFormatError, match="width"):
        read_trace_header(p)
    p.write_bytes(b"EDG")
    with pytest.raises(TraceFormatError, match="truncated header"):
        read_trace_header(p)


def test_truncation_reports_missing_bytes(tmp_path):
    path = tmp_path / "trunc.edgt"
    write_trace(path, [[np.zeros((4, 4))] for _ in range(3)])
    data = path.read_bytes()
    path.write_bytes(data[:-40])
    with pytest.raises(TraceFormatError, match="40 bytes missing"):
        list(replay_trace(path))
    path.write_bytes(data + bytes(8))
    with pytest.raises(TraceFormatError, match="8 trailing bytes"):
        read_trace_header(path)


def test_shape_change_rejected_on_write(tmp_path):
    with pytest.raises(ValueError):
        write_trace(tmp_path / "x.edgt", [[np.zeros((2, 2))], [np.zeros((3, 2))]])


# ---- device replay and analysis

@pytest.mark.gpu
def test_replay_bit_identical_and_ids(tmp_path):
    path = tmp_path / "t.edgt"
    frames = trace_frames()
    write_trace(path, frames)
    back = list(replay_trace(path))
    assert len(back) == len(frames)
    for t, (orig, got) in enumerate(zip(frames, back)):
        assert [m.layer_id for m in got] == [0, 1, 2]
        assert all(m.iteration == t for m in got)
        for a, b in zip(orig, got):
            assert b.data.is_cuda
            assert np.array_equal(a, b.data.cpu().numpy())


@pytest.mark.gpu
def test_replay_streams_across_chunks(tmp_path, monkeypatch):
    """Frames larger than a pinned chunk and chunks spanning frame boundaries."""
    from paper_2511_10333_b200 import trace as tr
    monkeypatch.setattr(tr, "_CHUNK_BYTES", 1000)  # not a divisor of the 3584-byte frame
    rng = np.random.default_rng(3)
    frames = [[rng.standard_normal((20, 30)).astype(np.float32), rng.standard_normal((7, 16)).astype(np.float32)]
              for _ in range(9)]
    path = tmp_path / "c.edgt"
    write_trace(path, frames)
    for orig, got in zip(frames, replay_trace(path)):
        for a, b in zip(orig, got):
            assert np.array_equal(a, b.data.cpu().numpy())


@pytest.mark.gpu
def test_replay_rejects_nonfinite(tmp_path):
    path = tmp_path / "n.edgt"
    bad = np.zeros((4, 4), np.float32)
    bad[1, 2] = np.nan
    write_trace(path, [[np.ones((4, 4))], [bad]])
    it = replay_trace(path)
    next(it)
    with pytest.raises(ValueError, match="non-finite"):
        next(it)


@pytest.mark.gpu
@pytest.mark.parametrize("estimator", ["histogram", "gaussian"])
def test_analyze_matches_reference(tmp_path, estimator):
    path = tmp_path / "t.edgt"
    write_trace(path, trace_frames())
    out = tmp_path / estimator
    analyze_trace(path, estimator=estimator, alpha=TRACE_SPEC["alpha"], beta=TRACE_SPEC["beta"], seed=3,
                  window=TRACE_SPEC["window"], correlation_iterations=TRACE_SPEC["correlation_iterations"],
                  output_dir=out)
    gold = GOLD["runs"][estimator]
    # histograms: counts and edges bit-exact -> the CSV is byte-identical
    assert (out / "gradient_histograms.csv").read_text() == gold["gradient_histograms.csv"]
    # windows: entropy to fp64 reduction order
    h, rows = _rows((out / "entropy_windows.csv").read_text())
    gh, grows = _rows(gold["entropy_windows.csv"])
    assert h == gh and len(rows) == len(grows)
    for r, g in zip(rows, grows):
        assert r[0] == g[0] and r[2] == g[2]
        assert abs(float(r[1]) - float(g[1])) <= 1e-12
    # correlations: same pairs, fp64 Gram vs np.dot
    h, rows = _rows((out / "layer_correlations.csv").read_text())
    gh, grows = _rows(gold["layer_correlations.csv"])
    assert h == gh and [r[:3] for r in rows] == [g[:3] for g in grows]
    for r, g in zip(rows, grows):
        assert abs(float(r[3]) - float(g[3])) <= 1e-12


@pytest.mark.gpu
def test_analyze_deterministic_and_unit_correlations(tmp_path):
    rng = np.random.default_rng(0)
    frames = []
    for _ in range(4):
        base = rng.standard_normal((16, 16)).astype(np.float32)
        frames.append([base.copy() for _ in range(3)])
    path = tmp_path / "same.edgt"
    write_trace(path, frames)
    res = analyze_trace(path, window=2, alpha=0.5)
    assert res.correlations and all(abs(r[3] - 1.0) <= 1e-12 for r in res.correlations)
    again = analyze_trace(path, window=2, alpha=0.5)
    assert again.histograms == res.histograms and again.correlations == res.correlations
    assert [w.mean_entropy for w in again.windows] == [w.mean_entropy for w in res.windows]
