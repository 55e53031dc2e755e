"""Print the SASS of one kernel of libising.so: python tools/sass_fun.py <cubin-stem> <mangled-substring>"""
import re, subprocess, sys
stem, pat = sys.argv[1], sys.argv[2]
so = "/root/repo/paper_2311_09275_b200/lib/libising.so"
subprocess.run(["cuobjdump", "-xelf", f"{stem}.sm_100a.cubin", so], cwd="/tmp", capture_output=True)
dis = subprocess.run(["nvdisasm", "-c", f"/tmp/{stem}.sm_100a.cubin"], capture_output=True, text=True).stdout
out, on = [], False
for ln in dis.splitlines():
    if ln.startswith(".text."):
        on = pat in ln
        continue
    if on and (re.match(r"\s+/\*[0-9a-f]+\*/", ln) or ln.startswith(".L")):
        out.append(re.sub(r"^\s+", "", ln))
print("\n".join(out))
