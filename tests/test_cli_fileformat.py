"""LMDW feature files, path files and the CLI's host-only commands (CPU);
`align` / `compare` run on the GPU in tests/test_gpu_cli.py."""
import io
import struct

import numpy as np
import pytest

import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import cli, fileformat as F, metrics


def test_features_round_trip(tmp_path):
    X = L.FeatureSeries(np.random.default_rng(0).standard_normal((37, 5)).astype(np.float32), 21.5)
    p = tmp_path / "a.lmdw"
    F.save_features(X, p)
    raw = p.read_bytes()
    assert raw[:4] == b"LMDW" and len(raw) == 18 + 37 * 5 * 4
    assert struct.unpack_from("<HII", raw, 4) == (1, 37, 5)
    Y = F.load_features(p)
    assert np.array_equal(Y.frames, X.frames) and Y.frame_rate == 21.5


def test_feature_format_errors(tmp_path):
    p = tmp_path / "bad.lmdw"
    p.write_bytes(b"LMD")
    with pytest.raises(F.FormatError, match=r"shorter than header \(byte offset 3\)"):
        F.load_features(p)
    p.write_bytes(struct.pack("<4sHIIf", b"XXXX", 1, 1, 1, 43.0) + b"\0" * 4)
    with pytest.raises(F.FormatError, match="bad magic"):
        F.load_features(p)
    p.write_bytes(struct.pack("<4sHIIf", b"LMDW", 2, 1, 1, 43.0) + b"\0" * 4)
    with pytest.raises(F.FormatError, match=r"unsupported version 2 \(byte offset 4\)"):
        F.load_features(p)
    p.write_bytes(struct.pack("<4sHIIf", b"LMDW", 1, 2, 2, 43.0) + b"\0" * 12)
    with pytest.raises(F.FormatError, match=r"payload is 12 bytes, header implies 16 \(byte offset 18\)"):
        F.load_features(p)
    p.write_bytes(struct.pack("<4sHIIf", b"LMDW", 1, 1, 3, 43.0) + np.array([0, np.inf, 1], "<f4").tobytes())
    with pytest.raises(F.FormatError, match=r"non-finite values \(byte offset 22\)"):
        F.load_features(p)


def test_path_file_round_trip(tmp_path):
    path = np.array([(0, 0), (1, 1), (1, 2), (2, 3)])
    p = tmp_path / "p.txt"
    F.save_path(path, 3, 4, 43.0664, 1.25, "linmdtw", p)
    assert p.read_text().splitlines()[0] == "# M=3 N=4 fps=43.0664 cost=1.25 algo=linmdtw"
    q, meta = F.load_path(p)
    assert np.array_equal(q, path) and meta == {"M": 3, "N": 4, "fps": 43.0664, "cost": 1.25, "algo": "linmdtw"}
    p.write_text("# nonsense\n0,0\n")
    with pytest.raises(F.FormatError, match="bad path header"):
        F.load_path(p)
    with pytest.raises(L.PathValidationError):
        F.save_path([(0, 0), (2, 2)], 3, 3, 43.0, 0.0, "x", p)


def test_memreport_and_estimates(capsys):
    assert cli.main(["memreport", "--m-seconds", "10", "--n-seconds", "12"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "frames: M=431 N=517 (fps 43.06640625)"
    assert out[1].split()[:2] == ["textbook", str(431 * 517)]
    assert metrics.memory_estimate("linmdtw", 431, 517).cells == 6 * 431
    assert metrics.memory_estimate("fastdtw", 100, 200, delta=30).cells == 100 * 125
    assert metrics.format_bytes(1536) == "1.5 KiB (1.54 KB)"
    assert metrics.format_bytes(12) == "12 B (12 B)"
    with pytest.raises(L.InvalidInputError):
        metrics.memory_estimate("bogus", 1, 1)


def test_cli_invalid_input_exit_code(tmp_path, capsys):
    p = tmp_path / "bad.lmdw"
    p.write_bytes(b"nope")
    assert cli.main(["align", str(p), str(p)]) == 2
    assert "error:" in capsys.readouterr().err


def test_report_round_trip():
    r = L.DiscrepancyReport(np.array([0, 3, 44]), fps=43.0)
    buf = io.StringIO()
    metrics.save_report(r, buf, (0.023, 1.0))
    text = buf.getvalue().splitlines()
    assert text[:4] == ["# fps=43.0", "# count=3", "# thresholds_s=0.023,1.0", "# proportions=0.333333,0.666667"]
    back = metrics.load_report(io.StringIO(buf.getvalue()))
    assert list(back.errors) == [0, 3, 44] and back.fps == 43.0
