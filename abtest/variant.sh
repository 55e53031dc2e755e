#!/bin/bash
# Build a variant of libising.so into abtest/lib_<name>.so with extra nvcc flags (e.g. -D overrides).
# usage: bash abtest/variant.sh <name> [nvcc flags...]
name=$1; shift
cd "$(dirname "$0")/.." && python - "$name" "$@" <<'PY'
import subprocess, sys
sys.path.insert(0, "paper_2311_09275_b200")
import build
name, extra = sys.argv[1], sys.argv[2:]
out = f"abtest/lib_{name}.so"
r = subprocess.run([build.NVCC, *build.FLAGS, *extra, "-o", out, *build.sources()], capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr); sys.exit(1)
import re
m = re.search(r"k_csr_i8_ringILi3ELi\d+EEEvNS_11CsrI8ParamsEjj' for 'sm_100a'\n.*\n.*\n(.*)", r.stdout + r.stderr)
print(name, m.group(1) if m else "")
PY
