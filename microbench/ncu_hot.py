"""Top stall-sampled SASS lines of an ncu source-page CSV (gz) export (dev helper)."""
import csv, gzip, io, sys
path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(io.TextIOWrapper(gzip.open(path), "utf-8")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
iS, iA = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
body = [r for r in rows[hi + 1:] if len(r) > iA and r[iA].replace(".", "").isdigit()]
tot = sum(float(r[iA]) for r in body)
for r in sorted(body, key=lambda r: -float(r[iA]))[:top]:
    print("%6.1f%%  %s  %s" % (100 * float(r[iA]) / tot, r[0], r[iS][:90]))
