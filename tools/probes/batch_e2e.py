"""Where cfg4's end-to-end time goes: the C call on host buffers (H2D inside)
vs building the Python results, for pinned inputs."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_02734_b200 as L  # noqa: E402
from paper_2008_02734_b200 import _capi  # noqa: E402
from paper_2008_02734_b200.divide import _c_config, _result  # noqa: E402

pairs = bench.make_inputs("cfg4")
pin = [(torch.from_numpy(X).pin_memory().numpy(), torch.from_numpy(Y).pin_memory().numpy()) for X, Y in pairs]
cfg = L.LinMdtwConfig(precision=32)
ccfg = _c_config(cfg)
lib = _capi.load()
n = len(pin)
xp = (C.c_void_p * n)(*[a.ctypes.data for a, _ in pin])
yp = (C.c_void_p * n)(*[b.ctypes.data for _, b in pin])
Ms = (C.c_int64 * n)(*[a.shape[0] for a, _ in pin])
Ns = (C.c_int64 * n)(*[b.shape[0] for _, b in pin])
for rep in range(3):
    h = (C.c_void_p * n)()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _capi.check(lib.lmdtw_align_batch(_capi.get_device(), n, xp, Ms, yp, Ns, 12, C.byref(ccfg), _capi.MEM_HOST, h))
    t1 = time.perf_counter()
    res = [_result(C.c_void_p(h[q]), Ms[q], Ns[q], np.float32) for q in range(n)]
    t2 = time.perf_counter()
    for q in range(n):
        lib.lmdtw_result_free(C.c_void_p(h[q]))
    t3 = time.perf_counter()
    fs = [(L.FeatureSeries(a), L.FeatureSeries(b)) for a, b in pin]
    t4 = time.perf_counter()
    r2 = L.align_batch(fs, config=cfg)
    t5 = time.perf_counter()
    print(f"C call {1e3 * (t1 - t0):.1f} ms, results {1e3 * (t2 - t1):.1f} ms, free {1e3 * (t3 - t2):.1f} ms, "
          f"align_batch {1e3 * (t5 - t4):.1f} ms", flush=True)
os.environ["LMDTW_PHASES"] = "1"
h = (C.c_void_p * n)()
_capi.check(lib.lmdtw_align_batch(_capi.get_device(), n, xp, Ms, yp, Ns, 12, C.byref(ccfg), _capi.MEM_HOST, h))
