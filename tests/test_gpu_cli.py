"""The CLI end to end on the GPU (cli.py:32-101 of the reference): LMDW files in,
path files out, every aligner, then `compare`."""
import numpy as np
import pytest

import bench
import paper_2008_02734_b200 as L
from paper_2008_02734_b200 import cli, fileformat as F

pytestmark = pytest.mark.gpu


def test_cli_align_and_compare(tmp_path, capsys):
    X, Y = bench.make_inputs("cfg1")[0]  # the reference golden pair (BASELINE cfg1)
    a, b = tmp_path / "a.lmdw", tmp_path / "b.lmdw"
    F.save_features(L.FeatureSeries(X), a)
    F.save_features(L.FeatureSeries(Y), b)
    outs = {}
    for algo in ("linmdtw", "dtw", "fastdtw", "mrmsdtw"):
        out = tmp_path / f"{algo}.txt"
        assert cli.main(["align", str(a), str(b), "--algo", algo, "--progress", "--out", str(out)]) == 0
        text = capsys.readouterr()
        lines = dict(l.split(":", 1) for l in text.out.splitlines())
        path, meta = F.load_path(out)
        outs[algo] = (path, meta)
        assert meta["M"] == 1000 and meta["N"] == 1000 and meta["algo"] in (algo, "dtw")
        if algo in ("linmdtw", "dtw"):
            # BASELINE cfg1 golden: the reference's fp64 cost and path length
            assert meta["cost"] == 11.1431643162049 and len(path) == 1073
            assert lines["cost"].strip() == "11.143164"
        if algo == "linmdtw":
            assert "progress:" in text.err
            assert lines["cells processed"].strip() == "1501687"
    assert np.array_equal(outs["linmdtw"][0], outs["dtw"][0])
    rep = tmp_path / "rep.txt"
    assert cli.main(["compare", str(tmp_path / "fastdtw.txt"), str(tmp_path / "linmdtw.txt"),
                     "--out", str(rep)]) == 0
    printed = capsys.readouterr().out.splitlines()
    assert printed[0].startswith("<=") and rep.read_text().startswith("# fps=")
    got = L.discrepancy(outs["fastdtw"][0], outs["linmdtw"][0])
    assert len(rep.read_text().splitlines()) == 4 + len(got.errors)
