"""Stall samples per source line from an ncu '--page source --csv --print-source cuda,sass' dump
(development tool): python tools/ncu_lines.py dump.csv [top]"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = [r for r in rows if r and r[0] == "Line No"][0]
cols = {h: i for i, h in enumerate(hdr)}
stall_names = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
byline = collections.Counter(); reasons = collections.defaultdict(collections.Counter)
tot = 0; cur = None; fn = None
for r in rows:
    if r and r[0] == "File Path": fn = r[1].split('/')[-1]
    if len(r) > 2 and r[0].isdigit(): cur = (fn, int(r[0]), r[1].strip()[:70])
    if len(r) > 5 and r[0] == "" and r[2].startswith('0x') and r[4].isdigit():
        v = int(r[4]); tot += v; byline[cur] += v
        for s in stall_names:
            x = r[cols[s]]
            if x.isdigit(): reasons[cur][s] += int(x)
allr = collections.Counter()
for k in reasons: allr.update(reasons[k])
print("total", tot, "|", ", ".join(f"{s[6:]}={100*c/tot:.1f}%" for s, c in allr.most_common(8)))
for key, v in byline.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    top = ", ".join(f"{s[6:]}={100*c/v:.0f}%" for s, c in reasons[key].most_common(3))
    print(f"{100*v/tot:5.1f}% {key[0]}:{key[1]} {key[2]} | {top}")
