#!/usr/bin/env python
"""SASS opcode histograms of the hot kernels in libhogb200.so (static counts
per kernel instantiation), so the Blackwell-specific claims (256-bit
STG.E.ENL2.256 plane stores, DFMA-dominated scores, no TMA on the default
plane path) can be checked without rebuilding.
usage: python tools/sass_hist.py [lib] > profiles/r2/sass_opcodes.txt"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_1703_06256_b200/libhogb200.so"
# (label, mangled-name pattern): the variants the BASELINE configs run
KERNELS = [
    ("k_planes c2 (NW=4, lattice step 4, 4 cols/lane, register top row, row-bulk TMA stores)",
     r"k_planesILi4ELi2ELi4ELb1ELi0ELb0ELb1ELb1EE"),
    ("k_planes c2 without row-bulk stores (HOGB200_ROWBULK=0: per-thread st.global)",
     r"k_planesILi4ELi2ELi4ELb1ELi0ELb0ELb1ELb0EE"),
    ("k_planes c4 (NW=4, lattice step 8, 8 cols/lane)", r"k_planesILi4ELi1ELi8ELb1ELi0ELb0ELb0EE"),
    ("k_planes c5 (NW=9, 18 bins, lattice step 8)", r"k_planesILi9ELi1ELi4ELb1ELi0ELb0ELb0EE"),
    ("k_grad_bin_oct gray, 8 bins, counts (c1/c2: fp16x2 octant sign tests, no table gather)",
     r"k_grad_bin_octILi8ELb1EE"),
    ("k_grad_bin gray, 8 bins, counts (table gather: any other table)", r"k_grad_binILi1ELi2ELb1EE"),
    ("k_grad_bin RGB, 8 bins, counts", r"k_grad_binILi3ELi2ELb1EE"),
    ("k_scores_rows, byte grid, 8 bins (c1/c4)", r"k_scores_rowsILi1ELi\d+ELi8ELb1ELi4EE"),
    ("k_scores_rows, byte grid, 18 bins (c5)", r"k_scores_rowsILi1ELi\d+ELi18ELb1ELi4EE"),
    ("k_resize", r"k_resize"),
]

sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if m and cur:
        funcs[cur].append(m.group(2))
for label, pat in KERNELS:
    names = [n for n in funcs if re.search(pat, n)]
    for n in names[:3]:
        ops = funcs[n]
        base = collections.Counter(o.split(".")[0] for o in ops)
        full = collections.Counter(ops)
        print(f"== {label}\n   {n}\n   {len(ops)} instructions")
        print("   by opcode: " + ", ".join(f"{k} {v}" for k, v in base.most_common(18)))
        mem = {k: v for k, v in full.items() if k.split(".")[0] in
               ("STG", "LDG", "STS", "LDS", "UTMASTG", "UBLKCP", "SHFL", "DFMA", "DMUL", "DADD",
                "I2F", "F2I", "FRND")}
        print("   memory / FP64 forms: " + ", ".join(f"{k} {v}" for k, v in sorted(mem.items())))
