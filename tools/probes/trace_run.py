"""One cfg3 alignment with LMDTW_TRACE_FILE set (run on the GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench
import paper_2008_02734_b200 as L
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
X, Y = bench.make_inputs(cfg)[0]
os.environ.pop("LMDTW_TRACE_FILE", None)
L.linmdtw(X, Y, min_dim=500, precision=32)  # warm-up
os.environ["LMDTW_TRACE_FILE"] = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/trace.bin"
r = L.linmdtw(X, Y, min_dim=500, precision=32)
print("cells", r.cells_processed)
