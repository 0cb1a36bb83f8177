#!/usr/bin/env python3
"""List the innermost backward-branch loops of each kernel in a cuobjdump -sass dump
with their instruction count and mnemonic mix (loop bodies = instructions per unit)."""
import collections
import re
import sys


def loops(path, pat=""):
    txt = open(path).read()
    for f in re.split(r'\n\s+Function : ', txt)[1:]:
        name = f.split('\n')[0].strip()
        if pat not in name:
            continue
        ins = []
        for l in f.split('\n'):
            m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        pos = {a: i for i, (a, _) in enumerate(ins)}
        out = []
        for i, (a, t) in enumerate(ins):
            m = re.search(r'BRA\s+0x([0-9a-f]+)', t)
            if m:
                tgt = int(m.group(1), 16)
                if tgt <= a and tgt in pos:
                    body = ins[pos[tgt]:i + 1]
                    c = collections.Counter(re.sub(r'^@!?U?P\w+\s+', '', x).split()[0].split('.')[0] for _, x in body)
                    if c['ATOMS'] or c['LDS'] or c['STG']:
                        out.append((len(body), hex(tgt), dict(c.most_common(12))))
        print(name)
        for o in sorted(out, key=lambda x: -x[0])[:4]:
            print("   ", o)


if __name__ == "__main__":
    loops(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
