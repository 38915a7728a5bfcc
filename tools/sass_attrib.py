"""Attribute a kernel's executed SASS instructions to the source statements they
are inlined under.

usage: python tools/sass_attrib.py SRC.csv CUBIN FUNC_INDEX FILE LO HI [CALL_FILE CALL_LINE]
  SRC.csv     `ncu -i REP --page source --csv --print-source cuda,sass` of one launch
  CUBIN       `cuobjdump -xelf all lib.so` output holding the kernel
  FUNC_INDEX  the kernel's symbol index (cuobjdump -elf: "function: NAME(0x..)")
  FILE LO HI  attribute to the outermost frame in FILE between lines LO..HI
  CALL_*      optional: only instructions inlined under CALL_FILE:CALL_LINE
Per-PC counts come from ncu, inline stacks from `nvdisasm -gi`; the opcodes of
the two listings are checked to agree."""
import collections
import csv
import re
import subprocess
import sys

src_csv, cubin, fidx, fname, lo, hi = sys.argv[1:7]
lo, hi = int(lo), int(hi)
call = (sys.argv[7], int(sys.argv[8])) if len(sys.argv) > 8 else None
rows = list(csv.reader(open(src_csv)))
hdr, cnt = None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("File Path", "Function Name"):
        continue
    if len(r) > 3 and r[2].startswith("0x"):
        try:
            ins = int(r[hdr.index("Instructions Executed")] or 0)
        except ValueError:
            continue
        cnt.setdefault(int(r[2], 16), (ins, int(r[4] or 0), r[3]))
base = min(cnt)
dis = subprocess.run(["nvdisasm", "-fun", fidx, "-gi", cubin], capture_output=True,
                     text=True).stdout
stack, pending, inst = [], [], {}
for ln in dis.splitlines():
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        pending.append((m.group(1).split("/")[-1], int(m.group(2))))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        if pending:
            stack, pending = pending, []
        inst[int(m.group(1), 16)] = (m.group(2), stack)
bad = sum(1 for off, (txt, _) in inst.items()
          if base + off in cnt and txt.split()[0].lstrip("@!P0123456789 ").split(".")[0]
          not in cnt[base + off][2])
print(f"{len(inst)} SASS instructions, {bad} opcode mismatches with the ncu listing")
lines = open(next(p for p in [fname] if True)).read().split("\n") if "/" in fname else None
agg, tot = collections.Counter(), 0
for off, (txt, st) in inst.items():
    c = cnt.get(base + off, (0, 0, ""))[0]
    if call and call not in st:
        continue
    key = None
    for f, l in st:
        if f == fname.split("/")[-1] and lo <= l <= hi:
            key = l
    agg[key] += c
    tot += c
for k, v in agg.most_common(40):
    print(f"{100 * v / max(tot, 1):5.1f}%  line {k}")
