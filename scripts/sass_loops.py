"""Static per-iteration instruction counts of the loops of one device
function (nvdisasm with line info): python scripts/sass_loops.py OBJ FUNC_SUBSTR"""
import re
import subprocess
import sys
import tempfile

import os
obj, func = os.path.abspath(sys.argv[1]), sys.argv[2]
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=d, check=True, capture_output=True)
    cub = subprocess.run("ls *.cubin", shell=True, cwd=d, capture_output=True, text=True).stdout.split()[0]
    sass = subprocess.run(["nvdisasm", "--print-line-info", cub], cwd=d, capture_output=True, text=True).stdout
lines = sass.splitlines()
start = next(i for i, l in enumerate(lines) if l.rstrip().endswith(":") and func in l and l.startswith("$"))
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("$") and lines[i].rstrip().endswith(":")
            or lines[i].startswith(".text.")), len(lines))
instrs, labels, cur = [], {}, None
for l in lines[start:end]:
    m = re.match(r'\s*//## File ".*", line (\d+)', l)
    if m:
        cur = int(m.group(1))
        continue
    m = re.match(r"^(\.L_x_\d+):", l.strip())
    if m:
        labels[m.group(1)] = len(instrs)
        continue
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        instrs.append((m.group(2), cur))
print(f"{func}: {len(instrs)} instructions")
for i, (t, ln) in enumerate(instrs):
    m = re.search(r"BRA.*`\((\.L_x_\d+)\)", t)
    if m and m.group(1) in labels and labels[m.group(1)] <= i:
        body = instrs[labels[m.group(1)]: i + 1]
        lns = sorted(set(x[1] for x in body if x[1]))
        print(f"  loop {m.group(1)}: {len(body):4d} instrs  lines {lns[:14]}{' ...' if len(lns) > 14 else ''}")
