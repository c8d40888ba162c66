"""Finds predicated global loads whose destination register is rewritten (by a later
instruction under another predicate) before any read — the pattern that makes the
warp wait for the load at the rewrite (long-scoreboard stall). Tuning aid:
    cuobjdump -sass libsrk.so > lib.sass; python scripts/sass_waw.py lib.sass <mangled-name-substring>
"""
import re
import sys

text = open(sys.argv[1]).read().split("Function : ")
want = sys.argv[2]
for fn in text:
    name = fn.split("\n", 1)[0]
    if want not in name:
        continue
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", fn)
    for i, (addr, s) in enumerate(ins):
        m = re.match(r"(@!?U?P\d\s+)?LDG\S*\s+(R\d+)", s)
        if not m or not m.group(1):
            continue
        rd = m.group(2)
        for a2, s2 in ins[i + 1:i + 150]:
            srcs = s2.split(None, 2)
            if re.search(rf"\b{rd}\b", s2.split(",", 1)[1] if "," in s2 else ""):
                break  # read first: fine
            m2 = re.match(rf"(@!?U?P\d\s+)?\S+\s+{rd}\b", s2)
            if m2:
                print(name[:90], addr, s.strip()[:60], "->", a2, s2.strip()[:60])
                break
