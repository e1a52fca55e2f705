"""Extract one kernel's SASS from a .so/.cubin and histogram its opcodes.
usage: python tools/sass_fn.py LIB SUBSTRING [--dump]"""
import re, subprocess, sys
lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_x]+)*)", f)
    hist = {}
    for o in ops:
        hist[o] = hist.get(o, 0) + 1
    print("==", name, len(ops), "instructions")
    print("  ", ", ".join(f"{k}:{v}" for k, v in sorted(hist.items(), key=lambda kv: -kv[1])[:40]))
    if "--dump" in sys.argv:
        print(f)
