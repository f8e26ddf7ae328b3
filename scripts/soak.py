import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch, time
from paper_1803_09948_b200 import HfmmCuda
from paper_1803_09948_b200.workloads import sphere_points, charges
free0 = torch.cuda.mem_get_info()[0]
n = 200000
xyz, q = sphere_points(n, 1), charges(n, 1)
ref = None
for it in range(30):
    op = HfmmCuda(k=4.0, order=12 if it % 3 else 14)
    op.set_points(xyz if it % 2 == 0 else xyz[: n // 2])
    y = op.matvec(q if it % 2 == 0 else q[: n // 2])
    assert np.isfinite(y).all()
    if it % 6 == 0:
        if ref is None: ref = y.copy()
        else: assert np.abs(y - ref).max() < 1e-4 * np.abs(ref).max()
    del op
free1 = torch.cuda.mem_get_info()[0]
print("handles ok; device memory delta MB", (free0 - free1) / 1e6)
op = HfmmCuda(k=4.0, order=12); op.set_points(xyz)
q_dev = torch.from_numpy(np.stack([q.real, q.imag], 1).astype(np.float32)).cuda(); out = torch.empty_like(q_dev)
op.matvec_device(q_dev.data_ptr(), out.data_ptr()); op.sync(); first = out.clone()
t = time.time()
for _ in range(500): op.matvec_device(q_dev.data_ptr(), out.data_ptr())
op.sync(); dt = time.time() - t
d = (out - first).abs().max().item() / first.abs().max().item()
print("500 matvecs %.2f s, %.2f ms each, drift vs first %.2e" % (dt, dt * 2, d))
