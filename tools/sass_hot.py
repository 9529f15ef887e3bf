import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {n: i for i, n in enumerate(hdr)}
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
data.sort(key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
print("total samples", tot)
for r in data[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((int(r[idx[c]] or 0), c[6:]) for c in cols), reverse=True)[:3]
    print(f"{s:7d} {100*s/tot:5.1f}% {r[idx['Address']]:>6} {r[idx['Source']][:60]:60s} {top}")
