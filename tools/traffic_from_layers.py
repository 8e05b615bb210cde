"""profiles/traffic.json from a tools/ncu_layers.sh capture: DRAM bytes
(dram__bytes_read.sum + dram__bytes_write.sum) and duration summed over the
kernels of each layer's SECOND launch set (the first warms the plan caches).
usage: python tools/traffic_from_layers.py gpurun_out/TAG_ncu.csv gpurun_out/TAG_plain.log CAPTURE_NAME > profiles/traffic.json"""
import csv
import json
import sys
from collections import OrderedDict

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(csv_path):
    rows = [l for l in open(csv_path) if l.startswith('"')]
    per = OrderedDict()
    for r in csv.DictReader(rows):
        e = per.setdefault(r["ID"], {"kernel": r["Kernel Name"].split("(")[0].replace("void ", "").strip()})
        e[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * UNIT.get(r["Metric Unit"], 1.0)
    return list(per.values())


def groups(ls):
    out, cur = [], []
    for e in ls:
        cur.append(e)
        if e["kernel"].split("::")[-1].startswith("conv_"):
            out.append(cur)
            cur = []
    return out


def main(csv_path, log_path, capture):
    names = [l.split()[1] for l in open(log_path) if l.startswith("i8  ")]
    g = groups(launches(csv_path))
    res = {"note": ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) and gpu__time_duration.sum summed "
                    "over the kernels one layer launches (the stem: the one-launch space-to-depth + the conv "
                    "kernel), second of two launches, batch 256, from tools/ncu_layers.sh (ncu flushes caches "
                    "per kernel: an output still L2-resident at kernel end shows fewer write bytes)."),
           "capture": capture, "layers": {}}
    for i, n in enumerate(names):
        ks = g[2 * i + 1]
        res["layers"][n] = {
            "kernels": [k["kernel"] for k in ks],
            "dram_bytes_per_launch": int(sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)
                                             for k in ks)),
            "kernel_us_sum": round(sum(k.get("gpu__time_duration.sum", 0) for k in ks), 2),
            "round": 2, "capture": capture}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4])
