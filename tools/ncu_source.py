"""Hot SASS blocks of an ncu report by executed instructions and stall samples:
python tools/ncu_source.py <rep> [threshold] [first-line last-line]"""
import csv, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ie = hdr.index("Instructions Executed"); src = hdr.index("Source"); samp = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie]) for r in data)
print("total", tot)
blocks = []; cur = None
for idx, r in enumerate(data):
    c = int(r[ie])
    if cur is None or c != cur[1]:
        if cur: blocks.append(cur)
        cur = [idx, c, 1, r[src].strip()[:50], int(r[samp])]
    else:
        cur[2] += 1; cur[4] += int(r[samp])
blocks.append(cur)
for b in blocks:
    if b[1] * b[2] > tot * thr:
        print(f"line {b[0]:5d} exec/instr {b[1]:9d} x {b[2]:4d} = {b[1]*b[2]/tot*100:5.1f}%  samples {b[4]:5d}  {b[3]}")
if len(sys.argv) > 3:
    a, b = int(sys.argv[3]), int(sys.argv[4])
    for r in data[a:b]:
        print(f"{int(r[ie]):9d} {int(r[samp]):5d}  {r[src].strip()[:90]}")
