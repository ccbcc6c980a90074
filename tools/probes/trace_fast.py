"""Per-strip-bucket pace and finish times of LMDTW_TRACE_FILE launches (hybrid queue study)."""
import sys
import numpy as np
sys.path.insert(0, __file__.rsplit("/", 1)[0])
from trace_strips import launches  # noqa: E402
H = 128
for li, (P, I, T, leaf, B) in enumerate(launches(sys.argv[1])):
    if li > 2 or leaf:
        continue
    t0 = T[:, 0].min()
    a = I["strip"]; b = I["blk"]
    pp = P[I["pass"]]
    W = pp["tile_w"]; c0 = b * W
    cols = np.minimum(np.minimum(pp["N"] - 1, pp["kstop"] - a * H), c0 + W - 1) - c0 + 1
    run = (T[:, 1] - B) / 1e3
    wait = (B - T[:, 0]) / 1e3
    pace = run * 1e3 * 1.965 / (cols + 32)
    span = (T[:, 1].max() - t0) / 1e6
    print(f"launch {li}: span {span:.3f} ms, items {len(I)}")
    for lo, hi in [(0, 1), (1, 8), (8, 40), (40, 80), (80, 160), (160, 400), (400, 2000)]:
        m = (a >= lo) & (a < hi)
        if m.sum() == 0:
            continue
        end = (T[m, 1].max() - t0) / 1e3
        print(f"   strips [{lo},{hi}): {m.sum():5d} tiles pace med {np.median(pace[m]):4.0f} mean {pace[m].mean():4.0f}"
              f"  tile-wait mean {wait[m].mean():6.1f} us  last end {end:8.1f} us")
