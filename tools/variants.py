"""Debug: build variant libraries with -D overrides (tools/variants/<name>.so) for A/B timing runs.

usage: python tools/variants.py name1:-DA=1,-DB=2 name2:-DA=3 ...
then on the GPU: PHASE_LIB=tools/variants/name1.so python tools/phase_time.py 3 2
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2501_07056_b200 import _lib  # noqa: E402

out = os.path.join(ROOT, "tools", "variants")
os.makedirs(out, exist_ok=True)
cus = [p for p in _lib.sources() if p.endswith(".cu")]
procs = []
for spec in sys.argv[1:]:
    name, _, flags = spec.partition(":")
    defs = [f for f in flags.split(",") if f]
    procs.append(subprocess.Popen(["nvcc", *_lib.NVCC_FLAGS, *defs, "-o", os.path.join(out, name + ".so"), *cus]))
sys.exit(max([p.wait() for p in procs] + [0]))
