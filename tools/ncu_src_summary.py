"""Per-SASS-line summary of an ncu source-page CSV export (the section of
the launch with the most instructions): instruction share, stall-sample
share, shared wavefronts vs ideal.
usage: ncu -i rep --page source --csv --print-source sass -k regex:K > f.csv
       python tools/ncu_src_summary.py f.csv [min_share]"""
import csv
import sys


def sections(rows):
    out = []
    for r in rows:
        if r and r[0] == "Kernel Name":
            out.append({"name": r[1], "rows": []})
        elif out:
            out[-1]["rows"].append(r)
    return out


def main():
    rows = list(csv.reader(open(sys.argv[1], errors="replace")))
    thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
    best = None
    for sec in sections(rows):
        hdr = sec["rows"][0]
        ci = {h: i for i, h in enumerate(hdr)}
        data = []
        for r in sec["rows"][1:]:
            if len(r) < len(hdr) or not r[ci["Instructions Executed"]].isdigit():
                continue
            data.append((int(r[ci["Instructions Executed"]]),
                         float(r[ci["Warp Stall Sampling (All Samples)"]] or 0),
                         r[ci["Address"]][-5:], r[ci["Source"]].strip()[:78],
                         r[ci["L1 Wavefronts Shared"]],
                         r[ci["L1 Wavefronts Shared Ideal"]]))
        tot = sum(d[0] for d in data)
        if best is None or tot > best[0]:
            best = (tot, sec["name"], data)
    tot, name, data = best
    ts = sum(d[1] for d in data) or 1
    print(name)
    print("total warp instructions", tot, "stall samples", ts)
    for d in data:
        if d[0] > tot * thr or d[1] > ts * 0.01:
            print(f"{d[0] / tot:6.3f} {d[1] / ts:6.3f} {d[2]} {d[3]:78s} "
                  f"{d[4]}/{d[5]}")


if __name__ == "__main__":
    main()
