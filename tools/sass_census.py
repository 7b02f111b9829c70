"""Per-kernel SASS opcode census of libmagnus_b200.so (cuobjdump -sass): global load/store widths,
bulk async copies (UBLKCP), shared-memory atomics, FMA use -- the evidence for the data-path
claims in DESIGN.md.  Usage: sass_census.py [lib.so] > profiles/<round>_sass_census.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2501_07056_b200/libmagnus_b200.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
kern = None
counts = collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        kern = m.group(1)
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if kern and m:
        op = m.group(2)
        base = op.split(".")[0]
        if base in ("LDG", "STG", "LDS", "STS", "ATOMS", "ATOMG", "RED", "REDG", "UBLKCP", "UTMALDG", "LDGSTS", "DFMA", "DMUL",
                    "DADD", "MATCH", "SHFL", "BAR", "SYNCS", "STAS"):
            counts[kern][op] += 1
names = sorted(counts, key=lambda k: -sum(counts[k].values()))
for k in names:
    pretty = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    if not pretty.startswith(("mg::", "void mg::")):
        continue
    c = counts[k]
    print(pretty[:110])
    for op in sorted(c):
        print(f"    {op:28s} {c[op]}")
