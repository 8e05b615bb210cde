"""Per-launch table from an ncu --set full report (ncu -i X --page raw --csv).
usage: ncu -i rep.ncu-rep --page raw --csv > raw.csv; python tools/ncu_table.py raw.csv"""
import csv
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3),
        ("dram__bytes_read.sum", "DRAM rd MB", 1e-6),
        ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor %", 1),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", 1),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %", 1),
        ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM MB", 1e-6),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %", 1),
        ("smsp__inst_executed.sum", "warp inst M", 1e-6),
        ("launch__registers_per_thread", "regs", 1),
        ("launch__grid_size", "grid", 1)]


def unit_scale(unit, metric):
    u = unit.strip().lower()
    if metric == "gpu__time_duration.sum":
        return {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6,
                "second": 1e9, "s": 1e9}.get(u, 1.0)
    if metric.startswith("dram__bytes") or metric.startswith("l1tex__m_"):
        return {"byte": 1.0, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1.0)
    return 1.0


def main(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    print("| kernel | " + " | ".join(c[1] for c in COLS) + " |")
    print("|---" * (len(COLS) + 1) + "|")
    for r in data:
        name = r[ix["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").replace("tzcdev::", "")
        cells = []
        for m, _, sc in COLS:
            if m not in ix or not r[ix[m]].strip():
                cells.append("-")
                continue
            v = float(r[ix[m]].replace(",", "")) * unit_scale(units[ix[m]], m) * sc
            cells.append(f"{v:.2f}" if abs(v) < 1000 else f"{v:.0f}")
        print(f"| `{short}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
