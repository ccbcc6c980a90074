"""Where a small alignment's time goes (cfg1, cfg2): wall time per call through
the C ABI on device-resident inputs, and one call with LMDTW_HOST_TIMING."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2008_02734_b200 as L  # noqa: E402
from paper_2008_02734_b200 import _capi  # noqa: E402
from paper_2008_02734_b200.divide import _c_config  # noqa: E402

lib = _capi.load()
for name in sys.argv[1:] or ["cfg1", "cfg2"]:
    X, Y = bench.make_inputs(name)[0]
    prec = bench.CONFIGS[name]["prec"]
    ccfg = _c_config(L.LinMdtwConfig(precision=prec))
    dX, dY = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()

    def once():
        h = C.c_void_p()
        _capi.check(lib.lmdtw_align(0, C.c_void_p(dX.data_ptr()), X.shape[0], C.c_void_p(dY.data_ptr()),
                                    Y.shape[0], X.shape[1], C.byref(ccfg), _capi.MEM_DEVICE, _capi.PROGRESS_FN(),
                                    None, C.byref(h)))
        info = _capi.AlignInfo()
        lib.lmdtw_result_info(h, C.byref(info))
        lib.lmdtw_result_free(h)
        return info
    for _ in range(5):
        once()
    reps = 50 if name == "cfg1" else 10
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        info = once()
    dt = (time.perf_counter() - t) / reps
    print(f"{name}: {dt * 1e3:.3f} ms per alignment, {info.cells_processed / dt / 1e9:.1f} GCUPS, "
          f"{info.n_levels} levels, {info.gpu_launches} launches", flush=True)
    os.environ["LMDTW_PHASES"] = "1"
    once()
    del os.environ["LMDTW_PHASES"]
