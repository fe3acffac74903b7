"""Opcode histogram of the timed loop (between the two clock reads) per kernel in a cuobjdump -sass dump."""
import collections
import re
import sys

FMAH = ("IMAD", "IMUL")
cur = None
d = {}
for line in open(sys.argv[1]):
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1); d[cur] = []; continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", line)
    if cur and m:
        d[cur].append(m.group(1).strip())
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
for k, body in d.items():
    idx = [i for i, x in enumerate(body) if "CLOCK" in x]
    b = body[idx[0]:idx[-1]] if len(idx) >= 2 else body
    c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] for x in b)
    wide = sum(v for o, v in c.items() if o.startswith("IMAD.WIDE") or o.startswith("IMAD.HI"))
    imad = sum(v for o, v in c.items() if o.startswith("IMAD") or o.startswith("IMUL")) - wide
    fp64 = sum(v for o, v in c.items() if o.split(".")[0] in ("DFMA", "DADD", "DMUL"))
    cv = sum(v for o, v in c.items() if o.split(".")[0] in ("I2F", "F2I"))
    alu = sum(v for o, v in c.items() if o.split(".")[0] in ("IADD3", "SEL", "ISETP", "LOP3", "SHF", "MOV", "PRMT", "LEA", "IADD"))
    print(f"{k}: n={len(b)/div:.2f} wide/hi={wide/div:.2f} imad={imad/div:.2f} fmaheavy_cyc~{(wide*5+imad*2)/div:.1f} alu={alu/div:.2f} (cyc {alu*2/div:.1f}) fp64={fp64/div:.2f} conv={cv/div:.2f}")
    print("    ", ", ".join(f"{o}:{v/div:.2f}" for o, v in sorted(c.items(), key=lambda t: -t[1])[:16]))
