import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from conftest import random_euclidean_matrix
import paper_1706_04399_b200 as pkg
rng = np.random.default_rng(31)
for n in (4, 5, 8, 16, 40, 100):
    cost = np.floor(random_euclidean_matrix(n, rng) * 100.0)
    tours = rng.permuted(np.tile(np.arange(n, dtype=np.int32), (6, 1)), axis=1)
    try:
        new, d = pkg.best_exchange_batch(cost, tours)
        print(n, "ok", d)
    except Exception as e:
        print(n, "ERR", e)
