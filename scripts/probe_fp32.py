"""GPU: scalar FFMA vs packed FFMA2 throughput probes (TFLOP/s)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_09948_b200 import HfmmCuda
op = HfmmCuda(k=1.0, order=4)
out = (ctypes.c_double * 2)()
for _ in range(3):
    rc = op.lib.hfmm_debug_fp32_probes(op.h, out)
    print("rc", rc, "FFMA %.2f TFLOP/s   FFMA2 %.2f TFLOP/s" % (out[0], out[1]))
