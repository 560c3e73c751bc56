"""Print the last call's kernels from an ncu --csv launch list (dev helper): name, duration, DRAM bytes."""
import csv, sys
from collections import OrderedDict
path, calls = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
h = rows[0]
i_n, i_m, i_v, i_id = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
k = OrderedDict()
for r in rows[1:]:
    k.setdefault(r[i_id], [r[i_n][:64], {}])[1][r[i_m]] = r[i_v]
items = list(k.values())
n = len(items) // calls
tot = 0.0
for name, v in items[-n:]:
    t = float(v.get("gpu__time_duration.sum", "0").replace(",", ""))
    tot += t
    print("  %-64s %10.0f ns  R %s W %s" % (name, t, v.get("dram__bytes_read.sum"), v.get("dram__bytes_write.sum")))
print("  total %.1f us over %d kernels" % (tot / 1e3, n))
