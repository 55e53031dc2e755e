"""Join ncu per-SASS-instruction execution counts with nvdisasm line info -> per source line."""
import csv, re, subprocess, sys
from collections import defaultdict

rep, cubin, fun = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line_of = {}
cur = None
insec = False
for ln in dis.splitlines():
    if ln.startswith("//----") and ".text." in ln:
        insec = ln.split(".text.")[1].split()[0] == fun
        continue
    if not insec:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f'{m.group(1).split("/")[-1]}:{m.group(2)}'
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]; data = rows[2:]
ia, ie, isrc = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
base = int(data[0][ia], 16)
per = defaultdict(int); tot = 0
for r in data:
    off = int(r[ia], 16) - base
    c = int(r[ie]); tot += c
    per[line_of.get(off, "?")] += c
src_cache = {}
def text(key):
    f, l = key.rsplit(":", 1)
    path = f"/root/repo/paper_2311_09275_b200/csrc/{f}"
    if path not in src_cache:
        try: src_cache[path] = open(path).read().splitlines()
        except OSError: src_cache[path] = []
    lines = src_cache[path]
    return lines[int(l) - 1].strip()[:70] if 0 < int(l) <= len(lines) else ""
print("total", tot)
for k, c in sorted(per.items(), key=lambda x: -x[1])[:top]:
    print(f"{c/tot*100:5.1f}% {k:26s} {text(k) if k != '?' else ''}")
