"""Stall-reason totals per kernel (and per source region) from a sass source CSV."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
i = 0
seen = set()
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Kernel Name":
        name = r[1]; hdr = rows[i + 1]; j = i + 2; body = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            body.append(rows[j]); j += 1
        if name not in seen:
            seen.add(name)
            cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
            tot = collections.Counter()
            for b in body:
                for c in cols:
                    tot[c[6:]] += int(b[hdr.index(c)] or 0)
            s = sum(tot.values())
            print("==", name[:90], s)
            print("   ", ", ".join(f"{k}={100*v/s:.1f}%" for k, v in tot.most_common(9)))
        i = j
    else:
        i += 1
