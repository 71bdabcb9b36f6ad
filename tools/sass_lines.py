"""Attribute ncu per-instruction counts to CUDA source lines.
usage: python tools/sass_lines.py <disasm from `nvdisasm -g`> <kernel mangled-name substring>
                                  <ncu --page source --csv --print-source sass output> [top]
Both listings are in address order; instruction i of one is instruction i of the other."""
import csv, re, sys, collections

dis, kname, ncsv = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines, cur, inside = [], None, False
for ln in open(dis):
    if ln.startswith("//-----") and ".text." in ln:
        inside = kname in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
rows = list(csv.reader(open(ncsv)))
h = rows[1]
ie, iS = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
data = rows[2:]
print(f"disasm instrs {len(lines)}, ncu instrs {len(data)}")
cnt, smp = collections.Counter(), collections.Counter()
for i, r in enumerate(data[: len(lines)]):
    cnt[lines[i]] += int(r[ie] or 0)
    smp[lines[i]] += int(r[iS] or 0)
tot, tots = sum(cnt.values()) or 1, sum(smp.values()) or 1
print(f"{'line':28s} {'instr%':>7s} {'samples%':>8s}")
for k, v in cnt.most_common(top):
    print(f"{str(k):28s} {100 * v / tot:7.2f} {100 * smp[k] / tots:8.2f}")
