"""Table from tools/sweep_layers.sh output: rows = layers, columns = variants (us, graph-replayed)."""
import sys

cur, tab, order = None, {}, []
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line[3:].strip() or "default"
        order.append(cur)
        continue
    p = line.split()
    if len(p) == 2:
        tab.setdefault(p[0], {})[cur] = float(p[1])
print("layer".ljust(20) + "".join(o.replace("--opt ", "")[:14].rjust(15) for o in order))
for k, v in tab.items():
    print(k.ljust(20) + "".join(f"{v.get(o, 0):15.1f}" for o in order))
