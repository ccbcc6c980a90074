"""Analyse LMDTW_TRACE_FILE dumps: per-strip DP start/end -> pace and waits."""
import sys
import numpy as np

PD = np.dtype([("x_off", "<i8"), ("y_off", "<i8"), ("M", "<i4"), ("N", "<i4"), ("kstop", "<i4"), ("reverse", "<i4"),
               ("rows", "<i4"), ("nstrips", "<i4"), ("out_off", "<i8", 6), ("bnd_off", "<i8"), ("bp_off", "<i8"),
               ("tab_off", "<i8"), ("bp_ld", "<i4"), ("leaf_id", "<i4"), ("lb_off", "<i8"),
               ("flag_off", "<i8"), ("tile_w", "<i4"), ("strip_lo", "<i4"), ("strip_hi", "<i4"),
               ("sys_out", "<i4"), ("bnd_in_first", "<u8"), ("win_first", "<i4"), ("win_count", "<i4")])
assert PD.itemsize == 168
WI = np.dtype([("pass", "<i4"), ("strip", "<i4"), ("blk", "<i4"), ("pad", "<i4")])


def launches(path):
    b = open(path, "rb").read()
    o = 0
    while o < len(b):
        npass, nit, leaf = np.frombuffer(b, "<i8", 3, o); o += 24
        P = np.frombuffer(b, PD, npass, o); o += PD.itemsize * npass
        I = np.frombuffer(b, WI, nit, o); o += WI.itemsize * nit
        T3 = np.frombuffer(b, "<u8", 3 * nit, o).reshape(-1, 3).astype(np.int64); o += 24 * nit
        T = T3[:, [0, 2]]; B = T3[:, 1]
        yield P, I, T, leaf, B


H = int(sys.argv[2]) if len(sys.argv) > 2 else 128
for li, (P, I, T, leaf, B) in enumerate(launches(sys.argv[1])):
    t0 = T[:, 0].min()
    dur = (T[:, 1] - T[:, 0]) / 1e3
    span = (T[:, 1].max() - t0) / 1e6
    a = I["strip"]; b = I["blk"]
    pp = P[I["pass"]]
    W = pp["tile_w"]
    c0 = b * W
    cols = np.minimum(np.minimum(pp["N"] - 1, pp["kstop"] - a * H), c0 + W - 1) - c0 + 1
    steps = cols + 32
    pace = dur * 1e3 * 1.965 / steps
    # busy fraction: sum of item durations / (span * number of pipelines)
    npipe = 592
    busy = dur.sum() / 1e3 / (span * npipe)
    print(f"launch {li} leaf={leaf} passes={len(P)} items={len(I)} span {span:.3f} ms busy {busy:.2f} "
          f"pace cyc/step: median {np.median(pace):.0f} p10 {np.percentile(pace, 10):.0f} p90 {np.percentile(pace, 90):.0f}")
    wait = (B - T[:, 0]) / 1e3
    run = (T[:, 1] - B) / 1e3
    rpace = run * 1e3 * 1.965 / steps
    print(f"   boundary wait: mean {wait.mean():.1f} us (b>0: {wait[b > 0].mean():.1f}); run pace median {np.median(rpace):.0f} "
          f"mean {np.average(rpace, weights=steps):.0f} p90 {np.percentile(rpace, 90):.0f}; wait share {wait.sum() / dur.sum():.2f}")
    if li == 0 or leaf:
        # time histogram of concurrently running items
        ts = np.linspace(0, span * 1e6, 21)
        conc = [int(((T[:, 0] - t0 <= t) & (T[:, 1] - t0 > t)).sum()) for t in ts]
        print("   running items over time:", conc)
        ends = (T[:, 1] - t0) / 1e3
        for q in np.argsort(ends)[-6:]:
            print(f"   late item pass {I['pass'][q]} strip {a[q]} blk {b[q]} start {(T[q,0]-t0)/1e3:.0f} us end {ends[q]:.0f} us "
                  f"dur {dur[q]:.0f} us steps {steps[q]} pace {pace[q]:.0f}")
