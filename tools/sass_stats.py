"""Per-kernel SASS statistics from `cuobjdump -sass` (offline, no GPU).

    python tools/sass_stats.py paper_2410_05934_b200/librnsntt.so [regex] [--full]

Prints, per matching kernel, the instruction count and an opcode histogram
(split into FMA-pipe IMAD family, ALU, memory, other) -- used to check the
per-butterfly instruction budget before spending GPU time.
"""
import collections
import re
import subprocess
import sys


def sections(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, []
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if cur:
                yield cur, body
            cur, body = m.group(1), []
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", line)
        if cur and m:
            body.append(m.group(1).strip())
    if cur:
        yield cur, body


def opcode(ins, full):
    ins = re.sub(r"^@!?U?P\w+\s+", "", ins)
    op = ins.split()[0]
    return op if full else op.split(".")[0]


def main():
    path = sys.argv[1]
    pat = re.compile(sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else ".")
    full = "--full" in sys.argv
    for name, body in sections(path):
        if not pat.search(name):
            continue
        c = collections.Counter(opcode(i, full) for i in body)
        fma = sum(v for k, v in c.items() if k.startswith("IMAD"))
        alu = sum(v for k, v in c.items() if k.split(".")[0] in ("IADD3", "ISETP", "SEL", "LOP3", "SHF", "LEA", "IABS", "IMNMX", "VIADD", "PRMT", "MOV"))
        mem = sum(v for k, v in c.items() if k.split(".")[0] in ("LDG", "STG", "LDS", "STS", "LDGSTS", "LD", "ST", "UBLKCP", "UTMALDG"))
        print(f"{name}: {len(body)} instrs  IMAD*={fma} ALU={alu} MEM={mem}")
        for k, v in c.most_common(40 if full else 25):
            print(f"    {v:6d} {k}")


if __name__ == "__main__":
    main()
