"""Per-source-line stall samples / executed instructions from an ncu report
(--page source --print-source=cuda,sass).  Usage: ncu_lines.py report.ncu-rep [file-substring]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
hdr = rows[hi]
ws, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
nidx = [hdr.index(n) for n in names]
cur_file, cur = "", None
agg = {}
for r in rows[:hi]:
    pass
for r in rows[hi + 1:]:
    if len(r) >= 2 and r[0] == "File Name":
        cur_file = r[1]
        continue
    if len(r) < 5:
        continue
    if r[0] and r[0].isdigit():
        cur = (cur_file.split("/")[-1], int(r[0]), r[1].strip()[:80])
        continue
    try:
        s, n = float(r[ws] or 0), float(r[ie] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0.0, 0.0, {}])
    a[0] += s
    a[1] += n
    for nm, i in zip(names, nidx):
        try:
            v = float(r[i] or 0)
        except ValueError:
            v = 0
        if v:
            a[2][nm] = a[2].get(nm, 0) + v
tot = sum(v[0] for v in agg.values())
print(f"total samples {tot:.0f}, warp insts {sum(v[1] for v in agg.values()):.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:30]:
    if k and want in k[0]:
        top = sorted(v[2].items(), key=lambda kv: -kv[1])[:3]
        print(f"{v[0]:6.0f} {v[1]:9.0f} {k[0]}:{k[1]} {k[2]} | " + " ".join(f"{a[6:]}={b:.0f}" for a, b in top))
