"""Build and run tools/gather_peaks.cu (the 2-opt scan's roofline peaks) and
write the JSON to profiles/<round>/gather_peaks.json.

    python tools/gather_peaks.py [--out profiles/r02/gather_peaks.json]

Peaks measured (see the .cu header): random fp64 gathers from L2-resident
(8-32 MB) and HBM tables, shared-memory gathers (random and conflict-free,
fp16 and fp64 elements), and the bulk-copy row stream L2 -> shared memory.
"""
import argparse
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02",
                                                  "gather_peaks.json"))
    args = ap.parse_args()
    build = os.path.join(ROOT, "build", "tools")
    os.makedirs(build, exist_ok=True)
    exe = os.path.join(build, "gather_peaks")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-std=c++17", "-lineinfo",
                           os.path.join(HERE, "gather_peaks.cu"), "-o", exe])
    if "--build-only" in sys.argv:
        return
    out = subprocess.check_output([exe]).decode()
    res = json.loads(out)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
