"""Aggregate `ncu --page source --print-source cuda,sass --csv` stall samples per CUDA source line."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
topn = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kern = None; hdr = None
out = collections.OrderedDict()
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        kern = r[1].split('(')[0].replace('void ', '')[:60] + ('|visc' if ', (bool)1' in r[1] else ''); out.setdefault(kern, []); continue
    if r and r[0] == "Line No": hdr = r; continue
    if not r or hdr is None or kern is None or not r[0].isdigit(): continue
    line = int(r[0]); src = r[1]
    samples = int(r[4]) if r[4].isdigit() else 0
    inst = int(r[7]) if r[7].isdigit() else 0
    stall = {h: int(v) for h, v in zip(hdr[29:46], r[29:46]) if v.isdigit()}
    out[kern].append((line, src.strip(), samples, inst, stall))
for k, v in out.items():
    tot = sum(x[2] for x in v) or 1
    print("=====", k, "total samples", tot)
    allst = collections.Counter()
    for x in v: allst.update(x[4])
    print("   overall:", [(a, f"{100*b/tot:.1f}%") for a, b in allst.most_common(7)])
    for line, src, s, inst, stall in sorted(v, key=lambda x: -x[2])[:topn]:
        top = [(a.replace('stall_', ''), b) for a, b in sorted(stall.items(), key=lambda kv: -kv[1])[:3]]
        print(f"{line:4d} {100*s/tot:5.1f}% inst={inst:10d} {src[:64]:64s} {top}")
