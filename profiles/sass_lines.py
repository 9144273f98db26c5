#!/usr/bin/env python3
"""Static SASS instruction count per source line of one kernel (nvdisasm -g output).

    cuobjdump -xelf all build/gbs_fp32.o; nvdisasm -g -c X.cubin > all.sass
    python profiles/sass_lines.py all.sass <kernel-substring> [file.cu]
"""
import re
import sys
from collections import Counter

path, kern = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else "gbs_fp32.cu"
cnt, cur, inside, total = Counter(), None, False, 0
for line in open(path):
    if line.startswith("//----") and ".text." in line:
        inside = kern in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = int(m.group(2)) if m.group(1).endswith(src) else None
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", line):
        total += 1
        cnt[cur] += 1
print("total", total)
for ln, c in sorted(cnt.items(), key=lambda t: -t[1])[:40]:
    print(ln, c)
