#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv --print-source sass` export by straight-line blocks
(consecutive SASS instructions with the same warp-execution count): share of thread
instructions and of warp-stall samples per block, and the stall totals by reason."""
import collections
import csv
import sys


def main(path, input_bytes):
    rows = list(csv.reader(open(path)))
    hdr, data = rows[1], rows[2:]
    iA, iS = hdr.index("Address"), hdr.index("Source")
    iT, iW = hdr.index("Thread Instructions Executed"), hdr.index("Instructions Executed")
    iSm = hdr.index("Warp Stall Sampling (All Samples)")
    stalls = [h for h in hdr if h.startswith("stall_") and "Not" not in h]
    data = [r for r in data if r[iT].isdigit()]
    tot = sum(int(r[iT]) for r in data)
    tots = sum(int(r[iSm] or 0) for r in data)
    print(f"# {rows[0][1]}")
    print(f"thread instructions {tot}  per input byte {tot / input_bytes:.3f}  warp-stall samples {tots}")
    st = collections.Counter()
    for r in data:
        for h in stalls:
            v = r[hdr.index(h)]
            if v.isdigit():
                st[h] += int(v)
    T = sum(st.values()) or 1
    print("stall reasons: " + ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in st.most_common(8)))
    print(f"{'addr':>6} {'warp-exec':>10} {'n':>4} {'thr-instr%':>10} {'samples%':>9}  first instruction / mix")
    cur = None
    out = []
    for r in data:
        w, t, sm = int(r[iW]), int(r[iT]), int(r[iSm] or 0)
        op = r[iS].strip().split()
        op = (op[1] if op and op[0].startswith("@") else (op[0] if op else "")).split(".")[0]
        if cur and cur["w"] == w:
            cur["t"] += t; cur["n"] += 1; cur["s"] += sm; cur["mix"][op] += 1
        else:
            if cur:
                out.append(cur)
            cur = {"a": r[iA][-5:], "src": r[iS].strip()[:40], "w": w, "t": t, "n": 1, "s": sm,
                   "mix": collections.Counter([op])}
    out.append(cur)
    for b in out:
        if b["t"] > 0.004 * tot or b["s"] > 0.01 * tots:
            mix = ",".join(f"{k}{v}" for k, v in b["mix"].most_common(5))
            print(f"{b['a']:>6} {b['w']:>10} {b['n']:>4} {100 * b['t'] / tot:>10.1f} {100 * b['s'] / tots:>9.1f}  {b['src']} | {mix}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
