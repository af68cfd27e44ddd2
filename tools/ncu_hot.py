"""Summarise an `ncu --page source --csv --print-source sass` dump: top SASS
lines by warp-stall samples with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
recs = []
for r in data:
    try:
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    tot += n
    top = sorted(((float(r[ix[s]] or 0), s) for s in stalls), reverse=True)[:3]
    recs.append((n, r[ix["Address"]], r[ix["Source"]][:60], top))
agg = {}
for r in data:
    for s in stalls:
        try:
            agg[s] = agg.get(s, 0) + float(r[ix[s]] or 0)
        except ValueError:
            pass
print("total samples", tot)
print("by reason:", ", ".join(f"{k[6:]}={v/tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for n, a, src, top in sorted(recs, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{n/tot:6.1%} {a} {src:60s} " + " ".join(f"{s[6:]}={v:.0f}" for v, s in top if v))
