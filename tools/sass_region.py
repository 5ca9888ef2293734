"""Print the SASS around the first occurrence of an opcode pattern:
    python tools/sass_region.py <sass.txt> <pattern> [before] [after]"""
import re
import sys

path, pat = sys.argv[1], sys.argv[2]
before = int(sys.argv[3]) if len(sys.argv) > 3 else 40
after = int(sys.argv[4]) if len(sys.argv) > 4 else 200
ins = []
for line in open(path):
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s*(.*?);", line)
    if m:
        ins.append((m.group(1), m.group(2).strip()))
idx = [k for k, (_, t) in enumerate(ins) if re.search(pat, t)]
if not idx:
    sys.exit("no match")
for a, t in ins[max(0, idx[0] - before):idx[0] + after]:
    print(a, t)
