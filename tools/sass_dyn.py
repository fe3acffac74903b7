"""Dynamic SASS opcode histogram from an ncu source-page export
(`ncu -i rep --page source --csv --print-source sass`): instructions executed
per opcode, and the fmaheavy-pipe cycle estimate (IMAD.WIDE / IMAD.HI 4 cycles
per warp instruction, other IMAD forms 2), normalised per `unit` (e.g. the
butterflies per launch).

    python tools/sass_dyn.py gpurun_out/sass/kw_sass.csv [butterflies]
"""
import collections
import csv
import re
import sys


def kernels(path):
    name, rows, hdr = None, [], None
    for r in csv.reader(open(path)):
        if len(r) >= 2 and r[0] == "Kernel Name":
            if name:
                yield name, rows
            name, rows, hdr = r[1], [], None
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            rows.append(dict(zip(hdr, r)))
    if name:
        yield name, rows


def main():
    path = sys.argv[1]
    unit = float(sys.argv[2]) if len(sys.argv) > 2 else None
    for name, rows in kernels(path):
        c = collections.Counter()
        stall = collections.Counter()
        tot = 0
        for d in rows:
            ins = re.sub(r"^@!?U?P\w+\s+", "", d["Source"].strip())
            op = ins.split()[0] if ins else "?"
            n = int(d["Instructions Executed"] or 0)
            c[op] += n
            tot += n
        wide = sum(v for o, v in c.items() if o.startswith("IMAD.WIDE") or o.startswith("IMAD.HI"))
        imad = sum(v for o, v in c.items() if (o.startswith("IMAD") or o.startswith("IMUL"))) - wide
        fmah = 4 * wide + 2 * imad
        print(f"== {name[:110]}")
        print(f"   warp instrs {tot:.4g}; fmaheavy warp-cycles ~{fmah:.4g}" + (f"; per unit: instrs {tot/unit:.2f}, fmaheavy {fmah/unit:.2f}" if unit else ""))
        for o, v in c.most_common(40):
            print(f"   {o:28s} {v:12d}" + (f"  {v/unit:7.3f}/unit" if unit else ""))


if __name__ == "__main__":
    main()
