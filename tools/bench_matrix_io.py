"""Plain-text matrix I/O: the native writer/reader
against the reference's Python (restated in oracle/graph_oracle.py) on an
N x N random-Euclidean matrix; checks byte identity and equal values.
Usage: python tools/bench_matrix_io.py [N]"""
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1706_04399_b200 as pkg  # noqa: E402
from oracle import graph_oracle as G  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    rng = np.random.default_rng(1)
    pts = rng.random((n, 2)) * 10
    c = np.sqrt(((pts[:, None] - pts[None]) ** 2).sum(-1))
    d = tempfile.mkdtemp()
    a, b = os.path.join(d, "ref.txt"), os.path.join(d, "ours.txt")
    t = time.perf_counter(); G.save_cost_matrix(a, c); s_ref = time.perf_counter() - t
    t = time.perf_counter(); pkg.save_cost_matrix(b, c); s_ours = time.perf_counter() - t
    same = open(a, "rb").read() == open(b, "rb").read()
    t = time.perf_counter(); x = G.load_cost_matrix(a); l_ref = time.perf_counter() - t
    t = time.perf_counter(); y = pkg.load_cost_matrix(a); l_ours = time.perf_counter() - t
    out = {"n": n, "bytes": os.path.getsize(a), "cores": os.cpu_count(),
           "save_ref_s": s_ref, "save_ours_s": s_ours, "save_identical": same,
           "load_ref_s": l_ref, "load_ours_s": l_ours,
           "load_equal": bool(np.array_equal(x, y))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
