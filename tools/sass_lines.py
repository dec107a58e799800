"""Per-source-line instruction counts / stall samples of one kernel: an ncu SASS page CSV
(`ncu -i rep --page source --csv --print-source sass`) joined with the line info of the
same build's SASS (`nvdisasm -g -c <cubin>`).  usage: sass_lines.py sass.csv all.sass mangled [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
body = rows[2:]
ia, ie, iw = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(body[0][ia], 16)
fn = sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
line_of = {}
cur = None
inside = False
for ln in open(sys.argv[2]):
    if ln.startswith(".text.") or ln.startswith("\t.section"):
        inside = fn in ln and ln.startswith(".text.")
        if ln.startswith(".text.") and fn not in ln:
            inside = False
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        line_of[int(m.group(1), 16)] = cur
ins = collections.Counter()
st = collections.Counter()
for r in body:
    off = int(r[ia], 16) - base
    k = line_of.get(off, "?")
    ins[k] += int(r[ie] or 0)
    st[k] += int(r[iw] or 0)
T, S = sum(ins.values()), sum(st.values())
print(f"total warp-instructions {T}, stall samples {S}")
for k, v in sorted(ins.items(), key=lambda x: -x[1])[:top]:
    print(f"{k:28s} {v:12d} {100 * v / T:5.1f}%  stall {100 * st[k] / max(S, 1):5.1f}%")
