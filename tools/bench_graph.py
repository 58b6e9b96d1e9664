"""Cost-matrix build benchmark on an office-sized grid.

Synthetic office-like occupancy in the shape of SURVEY §9 C2 (100x48x32
voxels: boundary walls, two pillars, a partition wall with a doorway and
desk blocks; unit axis weights) and 816 free viewpoint voxels from
default_rng(816).  Times ``build_cost_matrix`` on the device (CUDA events
around the ABI call, warm-up first) and checks sampled rows bit-exact
against the CPU Dijkstra oracle (integer weights: A* = Dijkstra bit for
bit).  The CPU time is the oracle's single-source Dijkstra on one core, per
source, times n; the reference's own pairwise A* (SURVEY: ~641 ms/pair on
this grid size, ~59 h for n=816) is far slower and cannot run on the box.

Usage: python tools/bench_graph.py [--n 816] [--reps 3] [--check 2]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def office_grid(nx=100, ny=48, nz=32):
    occ = np.zeros((nx, ny, nz), dtype=bool)
    occ[0, :, :] = occ[-1, :, :] = True
    occ[:, 0, :] = occ[:, -1, :] = True
    occ[:, :, 0] = True                      # floor
    for cx, cy in ((30, 20), (70, 28)):      # pillars, inflated
        occ[cx - 3:cx + 3, cy - 3:cy + 3, :] = True
    occ[50, 1:-1, 1:24] = True               # partition wall ...
    occ[50, 20:28, 1:18] = False             # ... with a doorway
    rng = np.random.default_rng(7)
    for _ in range(24):                      # desks
        x = int(rng.integers(3, nx - 10))
        y = int(rng.integers(3, ny - 8))
        occ[x:x + 6, y:y + 3, 1:4] = True
    return occ


def viewpoints(occ, n, seed=816):
    free = np.argwhere(~occ)
    rng = np.random.default_rng(seed)
    idx = rng.choice(len(free), size=n, replace=False)
    return free[np.sort(idx)].astype(np.int32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=816)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check", type=int, default=2)
    args = ap.parse_args()

    import torch
    from paper_1706_04399_b200 import build_cost_matrix
    from oracle import graph_oracle as G

    occ = office_grid()
    vox = viewpoints(occ, args.n)
    w = (1.0, 1.0, 1.0)
    build_cost_matrix(occ, vox, w)  # warm-up (module load, allocator)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        cost, virt, vcost = build_cost_matrix(occ, vox, w)
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / 1e3)
    gpu_s = float(np.median(times))

    # parity: rows of sampled sources vs the Dijkstra oracle (bit-exact for
    # integer weights); cost[i][j] is computed from min(i, j), so check i's
    # row to every j > i
    rng = np.random.default_rng(1)
    srcs = sorted(int(i) for i in rng.choice(args.n - 1, args.check,
                                             replace=False))
    cpu_t = []
    ok = True
    for i in srcs:
        t0 = time.perf_counter()
        d = G.dijkstra_all(occ, w, vox[i])
        cpu_t.append(time.perf_counter() - t0)
        for j in range(i + 1, args.n):
            want = d.get(tuple(int(c) for c in vox[j]))
            if want is None:
                ok &= bool(virt[i, j]) and cost[i, j] == vcost
            else:
                ok &= (not virt[i, j]) and cost[i, j] == want
    cpu_src = float(np.mean(cpu_t))
    V = occ.size
    print(json.dumps({
        "metric": "cost-matrix build time (all pairs)",
        "value": gpu_s, "unit": "s", "higher_is_better": False,
        "config": {"workload": "synthetic office grid 100x48x32, "
                   f"{args.n} viewpoints, unit weights",
                   "voxels": V, "free": int((~occ).sum()), "n": args.n},
        "parity_rows_checked": srcs, "parity_bit_exact": bool(ok),
        "virtual_pairs": int(virt.sum() // 2),
        "cpu_baseline": {"value": cpu_src * args.n, "unit": "s",
                         "cores": 1, "kind": "port",
                         "sample": f"{args.check} single-source Dijkstra "
                         f"runs ({cpu_src:.2f} s each) x n sources"},
        "reference_pairwise_astar_extrapolated_s":
            0.641 * args.n * (args.n - 1) / 2,
        "gpu_reps_s": times,
    }))


if __name__ == "__main__":
    main()
