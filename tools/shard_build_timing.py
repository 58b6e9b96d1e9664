"""Sharded cost-matrix build timed on one GPU: the one-call
build of a scene against each of W source shards (dpso_build_cost_rows)
run one after the other, plus the assemble step.  On W GPUs the SSSP phase
takes the slowest shard's time; the row all-gather moves n*n*8 bytes
(not measured here: one GPU).

    python tools/shard_build_timing.py office 8 > profiles/r02/shard_build_office.json
"""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_1706_04399_b200 import _lib, build_cost_matrix  # noqa: E402
from paper_1706_04399_b200.graph import _grid_args, source_blocks  # noqa


def timed(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "office"
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    occ, vox, w = scenes.scene(name)
    build_cost_matrix(occ, vox[:8], w)     # warm-up (module load, pools)
    one, t_one = timed(lambda: build_cost_matrix(occ, vox, w))
    o, v, wt = _grid_args(occ, vox, w)
    n = len(v)
    lib = _lib.load()
    docc = torch.from_numpy(o.ravel()).cuda()
    B, blocks = source_blocks(n, world)
    parts, shard_s = [], []
    for lo, hi in blocks:
        blk = torch.zeros((B, n), dtype=torch.float64, device="cuda")
        _, t = timed(lambda: _lib.check(lib.dpso_build_cost_rows(
            docc.data_ptr(), *o.shape, wt.ctypes.data_as(ctypes.c_void_p),
            v.ctypes.data_as(ctypes.c_void_p), n, lo, hi, blk.data_ptr(),
            None)))
        parts.append(blk)
        shard_s.append(t)
    rows = torch.cat(parts)[:n].contiguous()
    ld = (n + 7) // 8 * 8
    cost = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    virt = torch.zeros((n, n), dtype=torch.uint8, device="cuda")
    vc = ctypes.c_double()
    _, t_asm = timed(lambda: _lib.check(lib.dpso_build_cost_assemble(
        rows.data_ptr(), n, cost.data_ptr(), ld, virt.data_ptr(),
        ctypes.byref(vc), None)))
    same = bool(np.array_equal(cost[:, :n].cpu().numpy(), one[0])
                and vc.value == one[2])
    print(json.dumps({
        "scene": name, "grid": list(occ.shape), "n": n, "world": world,
        "one_call_s": round(t_one, 4),
        "shard_s": [round(t, 4) for t in shard_s],
        "slowest_shard_s": round(max(shard_s), 4),
        "assemble_s": round(t_asm, 5),
        "gather_bytes": n * n * 8,
        "identical_to_one_call": same,
        "note": "shards run one after the other on one GPU; on W GPUs the "
                "SSSP phase is the slowest shard, then one all-gather of "
                "gather_bytes over NVLink"}))


if __name__ == "__main__":
    main()
