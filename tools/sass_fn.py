"""Print the SASS of the functions whose name contains a substring:
    python tools/sass_fn.py <lib.so> <substring> [--stats]"""
import subprocess
import sys
from collections import Counter

lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in out.splitlines():
    if "Function : " in line:
        cur = line.split("Function : ")[1].strip()
        funcs[cur] = []
    elif cur:
        funcs[cur].append(line)
for name, lines in funcs.items():
    if pat not in name:
        continue
    ins = [l for l in lines if "/*" in l and ";" in l]
    print(f"== {name}: {len(ins)} instructions")
    if "--stats" in sys.argv:
        ops = Counter(l.split(";")[0].split("*/")[1].strip().split()[0].lstrip("@!P0123456789T ")
                      .split(".")[0] if "*/" in l else "" for l in ins)
        print(ops.most_common(40))
    else:
        print("\n".join(lines))
