"""Per-layer table from tools/ncu_layers.sh: ncu --csv (one row per metric per
launch) + the plain run's plan log (one line per layer, in launch order).
Each layer launches its kernels twice; the second launch set is reported."""
import csv
import sys
from collections import OrderedDict



def main(csv_path, log_path):
    names = [l.split()[1] for l in open(log_path) if l.startswith("i8  ")]
    rows = [l for l in open(csv_path) if l.startswith('"')]
    per = OrderedDict()
    for r in csv.DictReader(rows):
        key = r["ID"]
        e = per.setdefault(key, {"kernel": r["Kernel Name"].split("(")[0].replace("void ", "").strip()})
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
                 "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
                 "Gbyte": 1e3, "%": 1.0}.get(u, 1.0)
        e[r["Metric Name"]] = v * scale
    L = list(per.values())
    # group: a launch of conv_* ends a layer's kernel set (stem: s2d, weights, conv)
    groups, cur = [], []
    for e in L:
        cur.append(e)
        if e["kernel"].split("::")[-1].startswith("conv_") or "splitk" in e["kernel"]:
            if "splitk" in e["kernel"] and groups and cur == [e]:
                groups[-1].append(e)
                cur = []
                continue
            groups.append(cur)
            cur = []
    print("| layer | kernels | us | DRAM rd MB | DRAM wr MB | tensor % | issue % | L2 MB |")
    print("|---|---|---|---|---|---|---|---|")
    tot = 0.0
    for i, name in enumerate(names):
        g = groups[2 * i + 1] if 2 * i + 1 < len(groups) else []
        us = sum(e.get("gpu__time_duration.sum", 0) for e in g)
        tot += us
        rd = sum(e.get("dram__bytes_read.sum", 0) for e in g)
        wr = sum(e.get("dram__bytes_write.sum", 0) for e in g)
        lt = sum(e.get("lts__t_bytes.sum", 0) for e in g)
        conv = g[-1] if g else {}
        print(f"| {name} | {len(g)} | {us:.2f} | {rd:.1f} | {wr:.1f} | "
              f"{conv.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
              f"{conv.get('sm__inst_issued.avg.pct_of_peak_sustained_elapsed', 0):.1f} | {lt:.1f} |")
    print(f"\nsum of layer kernels: {tot:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
