"""Opcode histogram (dynamic, from an ncu `--page source --csv --print-source sass`
export): instructions executed and stall samples per SASS opcode, per kernel."""
import collections
import csv
import sys


def blocks(path):
    cur = None
    for ln in open(path).read().split("\n"):
        if ln.startswith('"Kernel Name"'):
            if cur:
                yield cur
            cur = [ln]
        elif cur is not None:
            cur.append(ln)
    if cur:
        yield cur


def main(path, top=25):
    for b in blocks(path):
        name = next(csv.reader([b[0]]))[1]
        rows = list(csv.reader(b[1:]))
        hdr = rows[0]
        ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
        st = hdr.index("Warp Stall Sampling (All Samples)")
        ops, stalls, tot = collections.Counter(), collections.Counter(), 0
        for r in rows[1:]:
            if len(r) <= ie or not r[ie].isdigit():
                continue
            n = int(r[ie])
            toks = r[src].split()
            if not toks:
                continue
            op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
            ops[op] += n
            stalls[op] += int(r[st] or 0)
            tot += n
        print(f"== {name}\ninstructions executed (warp-level): {tot}")
        for op, n in ops.most_common(top):
            print(f"  {op:10s} {n:12d} {100.0 * n / tot:5.1f}%  stall-samples {stalls[op]}")


if __name__ == "__main__":
    main(sys.argv[1])
