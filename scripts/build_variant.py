"""Builds the CUDA library with extra -D defines into _lib/variants/<name>.so (A/B
development aid; load one with SG_LIB_OVERRIDE=<path>).
usage: build_variant.py name -DSG_BAND_R=4 -DSG_CWARPS=2 ..."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2208_09985_b200 import build as b
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.LIB_DIR, "variants", name + ".so")
os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = [b.nvcc(), *b.NVCC_FLAGS, *defs, "-shared", "-o", out,
       *[os.path.join(b.CSRC, f) for f in b.SOURCES], "-lpthread"]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stderr)
    sys.exit(1)
for line in r.stderr.splitlines():
    if "k1_mixedILi2" in line and "Compiling" in line:
        i = r.stderr.splitlines().index(line)
        print(name, " | ".join(x.strip() for x in r.stderr.splitlines()[i + 1:i + 3]))
print(out)
