#!/bin/bash
# rebuild libsetbwte.so (sm_100a) in-tree and show register/stack use per kernel
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0,'.')
from paper_1410_0562_b200 import _build; _build.build()" || exit 1
python - <<'PY'
import glob, re
for f in sorted(glob.glob('build/*.ptxas.log')):
    name = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m: name = m.group(1)
        if 'error' in line or 'warning' in line: print(line.rstrip())
        m = re.search(r"Used (\d+) registers.*?(\d+) bytes cumulative stack size(.*)", line)
        if m and name: print("%-60s regs=%s stack=%s %s" % (name[:60], m.group(1), m.group(2), m.group(3).strip()))
PY
