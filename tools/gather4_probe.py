"""Build and run tools/gather4_probe.cu (bulk row copies vs TMA gather4 into
shared memory) and write profiles/r02/gather4_probe.json.

    python tools/gather4_probe.py [--out ...]
"""
import argparse
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02",
                                                  "gather4_probe.json"))
    args = ap.parse_args()
    build = os.path.join(ROOT, "build", "tools")
    os.makedirs(build, exist_ok=True)
    exe = os.path.join(build, "gather4_probe")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-O3", "-std=c++17", "-lineinfo",
                           os.path.join(HERE, "gather4_probe.cu"), "-o", exe])
    res = json.loads(subprocess.check_output([exe], timeout=300).decode())
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
