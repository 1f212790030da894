"""Markdown summary of ncu --set full captures (one kernel launch each):
duration, DRAM bytes read / written, DRAM and L2 throughput, hit rates,
occupancy, issue activity and the top warp-stall reasons.

    python tools/ncu_report.py label=report.ncu-rep [...] > profiles/rNN_xxx.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, r)} for r in rows[2:]]


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def main():
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " | top stall samples |")
    print("|---" * (len(METRICS) + 2) + "|")
    for arg in sys.argv[1:]:
        label, rep = arg.split("=", 1)
        for r in raw(rep):
            cells = []
            for key, _ in METRICS:
                v, u = r.get(key, ("", ""))
                cells.append(f"{v} {u}".strip())
            stalls = []
            pre = "smsp__pcsamp_warps_issue_stalled_"
            for k, (v, u) in r.items():
                if k.startswith(pre) and not k.endswith("_not_issued"):
                    x = num(v)
                    if x:
                        stalls.append((x, k[len(pre):]))
            tot = sum(x for x, _ in stalls) or 1.0
            stalls.sort(reverse=True)
            st = ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in stalls[:4])
            name = r.get("Kernel Name", ("?", ""))[0][:40]
            print(f"| {label}: `{name}` | " + " | ".join(cells) + f" | {st} |")


if __name__ == "__main__":
    main()
