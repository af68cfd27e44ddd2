"""Print (kernel, duration) rows of an `ncu --metrics gpu__time_duration.sum --csv` log."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum" and pat in d["Kernel Name"]:
            print(f"{d['Kernel Name'][:70]:70s} {d['Metric Value']:>12s} {d['Metric Unit']}")
