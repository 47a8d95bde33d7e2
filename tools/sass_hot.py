"""Aggregate an ncu '--page source --csv --print-source sass' dump: stall samples by opcode and
the hottest instructions with context (development tool)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_src = hdr.index("Source"); i_a = hdr.index("Address")
val = lambda r: int(r[i_s]) if r[i_s].isdigit() else 0
tot = sum(val(r) for r in data)
by = collections.Counter()
for r in data:
    t = r[i_src].split()
    if not t: continue
    op = t[1] if t[0].startswith('@') else t[0]
    by[op.split('.')[0]] += val(r)
print("total samples", tot)
for k, v in by.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{k:12s} {v:9d} {100 * v / tot:5.1f}%")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
for k, r in sorted(enumerate(data), key=lambda kr: -val(kr[1]))[:n]:
    print(f"--- {100 * val(r) / tot:.1f}% at {r[i_a][-5:]}")
    for rr in data[max(0, k - 4):k + 2]:
        print(f"   {rr[i_a][-5:]} {val(rr):8d} {rr[i_src][:90]}")
