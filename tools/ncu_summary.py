"""One-line-per-launch summary of an ncu --set full report (raw page):
duration, DRAM bytes, shared wavefronts and bank conflicts, instructions,
issue utilisation, warps, registers.
usage: python tools/ncu_summary.py rep.ncu-rep [out.txt]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("gpc__cycles_elapsed.avg.per_second", "clock"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_thr_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts"),
    ("smsp__inst_executed.sum", "instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def main():
    raw = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "raw",
                                   "--csv"]).decode()
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    u = dict(zip(hdr, units))
    out = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        parts = [d.get("Kernel Name", "")[:60]]
        for k, name in KEYS:
            if k in d:
                parts.append(f"{name}={d[k]} {u.get(k, '')}".strip())
        out.append("  ".join(parts))
    text = "\n".join(out) + "\n"
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(text)
    print(text)


if __name__ == "__main__":
    main()
