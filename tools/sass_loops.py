"""Per-loop instruction mix of a kernel's SASS (cuobjdump -sass of one
function): every backward branch = one loop; prints its body size, FP64
instructions and the rest.  Usage: python tools/sass_loops.py OBJ MANGLED_SUBSTR"""
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ins = []
    for line in f.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(name)
    for a, t in ins:
        mm = re.search(r"BRA\b.*?(0x[0-9a-f]+|`\(\.L_x_(\d+)\))", t)
        if not mm or not mm.group(1).startswith("0x"):
            continue
        tgt = int(mm.group(1), 16)
        if tgt >= a:
            continue
        body = [x for x in ins if tgt <= x[0] <= a]
        fp = sum(1 for x in body if re.search(r"\bD(ADD|MUL|FMA)\b", x[1]))
        print(f"  loop {tgt:#07x}..{a:#07x}: {len(body):3d} instr, {fp:3d} FP64, {len(body) - fp:3d} other")
