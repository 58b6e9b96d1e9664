"""Debug harness: band scan on n x P random tours vs the oracle (sampled)."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from conftest import random_euclidean_matrix
import paper_1706_04399_b200 as pkg
from oracle import dpso_oracle as O
n = int(os.environ.get("N", "500")); P = int(os.environ.get("P", "3000"))
kind = os.environ.get("KIND", "grid")
rng = np.random.default_rng(5)
if kind == "grid":
    import math
    side = int(math.ceil(math.sqrt(n))); idx = np.arange(n)
    pts = np.stack([idx % side, idx // side], 1).astype(float)
    cost = np.abs(pts[:, None, :] - pts[None, :, :]).sum(-1)
else:
    cost = random_euclidean_matrix(n, rng)
tours = rng.permuted(np.tile(np.arange(n, dtype=np.int32), (P, 1)), axis=1)
new, d = pkg.best_exchange_batch(cost, tours)
bad = 0
for p in rng.choice(P, size=min(P, 40), replace=False):
    eb, ed = O.best_exchange([int(v) for v in tours[p]], cost)
    if list(map(int, new[p])) != list(map(int, eb)) or float(d[p]) != ed:
        bad += 1
print("n", n, "P", P, "bad", bad)
print("nan deltas", int(np.isnan(d).sum()))
