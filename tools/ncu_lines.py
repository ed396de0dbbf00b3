"""Per-source-line instruction / stall breakdown of an .ncu-rep captured with --import-source on."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; fname = None; agg = []; cur = None
for r in rows:
    if len(r) >= 2 and r[0] == 'File Path': fname = r[1].split('/')[-1]; continue
    if r and r[0] == 'Line No': hdr = r; continue
    if hdr is None or len(r) < len(hdr) - 5: continue
    if r[0] != '':
        try:
            cur = [fname, int(r[0]), r[1].strip(), int(r[7]), int(r[4]), {}]
            agg.append(cur)
        except ValueError:
            pass
    elif cur is not None:
        op = r[3].split()
        if op:
            name = op[1] if op[0].startswith('@') else op[0]
            name = name.split('.')[0]
            try: cur[5][name] = cur[5].get(name, 0) + int(r[7])
            except ValueError: pass
tot = sum(a[3] for a in agg); ts = sum(a[4] for a in agg)
print('total warp-inst', tot, 'stall samples', ts)
agg.sort(key=lambda a: -(a[4] if len(sys.argv) > 3 else a[3]))
for a in agg[:top]:
    ops = sorted(a[5].items(), key=lambda kv: -kv[1])[:4]
    print(f'{a[0]}:{a[1]:4d} {100*a[3]/tot:5.1f}% inst {100*a[4]/ts:5.1f}% stall  {a[2][:80]:80s} {" ".join(f"{k}:{100*v/tot:.1f}" for k,v in ops)}')
