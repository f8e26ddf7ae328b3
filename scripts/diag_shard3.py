import os, sys, ctypes
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.api import load_library
from paper_1803_09948_b200.distributed import emulate_gmres_on_one_device
lib = load_library(); lib.hfmm_debug_stale_cuda_error.restype = ctypes.c_char_p
G = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "solver.npz"))
def mk(r, ranks):
    op = HfmmCuda(k=float(G["bie_k"]), order=int(G["bie_order"]), ncrit=16, theta=0.4, kd_max=1.0, leaf_cap=-1.0)
    op.set_partition(r, ranks)
    op.set_points(G["bie_xyz"])
    print("   stale after set_points:", lib.hfmm_debug_stale_cuda_error(), flush=True)
    op.set_corrections(int(G["bie_ni"]), far_weight=G["bie_far_weight"], patch_block=G["bie_patch_block"],
                       near_offset=G["bie_near_offset"], near_source=G["bie_near_source"],
                       near_delta=G["bie_near_delta"], block_lu=G["bie_block_lu"], block_piv=G["bie_block_piv"])
    return op
for ranks in (2, 3):
    ops = [mk(r, ranks) for r in range(ranks)]
    order = ops[0].body_order()
    res = emulate_gmres_on_one_device(ops, np.asarray(G["bie_rhs"])[order], rtol=1e-4, restart=30, max_iterations=200)
    print(ranks, [r[1]["iterations"] for r in res], "stale:", lib.hfmm_debug_stale_cuda_error(), flush=True)
    del ops, res
