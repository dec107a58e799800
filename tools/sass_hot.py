"""Top SASS instructions by warp-stall samples per kernel from `ncu --page source --csv --print-source sass`."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
i = 0
while i < len(rows):
    r = rows[i]
    if r and r[0] == "Kernel Name":
        name = r[1]
        hdr = rows[i + 1]
        j = i + 2
        body = []
        while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
            body.append(rows[j]); j += 1
        if want in name:
            si = hdr.index("Warp Stall Sampling (All Samples)")
            tot = sum(int(b[si] or 0) for b in body)
            print("==", name[:100], "samples", tot)
            cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
            ci = [hdr.index(c) for c in cols]
            for k, b in enumerate(body):
                b.append(k)
            ranked = sorted(body, key=lambda b: -int(b[si] or 0))[:top]
            for b in sorted(ranked, key=lambda b: b[-1]):
                st = sorted(((int(b[x] or 0), c[6:]) for x, c in zip(ci, cols)), reverse=True)[:3]
                print(f"{b[-1]:5d} {int(b[si] or 0):6d} {100*int(b[si] or 0)/max(tot,1):5.1f}%  {b[1].strip()[:60]:60s} {st}")
            want = "\x00"  # first match only
        i = j
    else:
        i += 1
