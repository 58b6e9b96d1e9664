"""Time the 2-opt scan kernels alone (batch API, random tours) at one size:
python tools/scan_probe.py N P  -> prints ms per batch call (CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1706_04399_b200 import _lib  # noqa: E402
from paper_1706_04399_b200.solver import device_cost  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
rng = np.random.default_rng(1)
pts = rng.random((n, 2)) * 10
cost = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
cdev, ld = device_cost(cost)
tours = torch.from_numpy(np.stack([rng.permutation(n) for _ in range(P)])
                         .astype(np.int32)).cuda()
delta = torch.empty(P, dtype=torch.float64, device="cuda")
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
def call():
    t = tours.clone()
    _lib.check(lib.dpso_best_exchange_batch(cdev.data_ptr(), ld, n, t.data_ptr(),
                                            P, delta.data_ptr(), st))
for _ in range(3):
    call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(5):
    call()
e1.record(); torch.cuda.synchronize()
print(f"n={n} P={P} mode={os.environ.get('DPSO_SCAN_MODE','auto')} stream_only={os.environ.get('DPSO_SCAN_STREAM_ONLY','0')}: {e0.elapsed_time(e1)/5:.3f} ms per batch call")
