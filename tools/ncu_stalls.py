"""Summarise an ncu --page source --csv --print-source sass dump: stall totals by
reason, and the top instructions with their dominant reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: sum(float(d[idx[r]] or 0) for d in data) for r in reasons}
allt = sum(tot.values())
print("total samples %.0f" % allt)
for r, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print("  %-24s %5.1f%%" % (r, 100 * v / allt))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
print("top instructions:")
for d in sorted(data, key=lambda d: -float(d[idx["Warp Stall Sampling (All Samples)"]] or 0))[:n]:
    rs = sorted(((r, float(d[idx[r]] or 0)) for r in reasons), key=lambda kv: -kv[1])[:2]
    print("  %-56s %7s  %s" % (d[idx["Source"]][:56], d[idx["Warp Stall Sampling (All Samples)"]],
                                " ".join("%s=%.0f" % (r[6:], v) for r, v in rs)))
