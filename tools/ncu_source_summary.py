"""Summarise `ncu --page source --csv --print-source sass` output by basic block
(instructions grouped by execution count): executed share, stall share, opcode mix."""
import csv
import sys
from collections import Counter, defaultdict


def sections(path):
    rows = list(csv.reader(open(path)))
    cur_name, hdr, data = None, None, []
    for r in rows:
        if r and r[0] == "Kernel Name":
            if hdr:
                yield cur_name, hdr, data
            cur_name, hdr, data = r[1], None, []
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and len(r) == len(hdr):
            data.append(r)
    if hdr:
        yield cur_name, hdr, data


for name, h, data in sections(sys.argv[1]):
    isrc, iex, ist = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    tot_ex = sum(int(r[iex]) for r in data) or 1
    tot_st = sum(int(r[ist]) for r in data) or 1
    print("==", name[:90], "executed", tot_ex, "samples", tot_st)
    groups = defaultdict(lambda: [0, 0, 0, []])
    for r in data:
        ex = int(r[iex])
        g = groups[ex]
        g[0] += 1
        g[1] += ex
        g[2] += int(r[ist])
        op = r[isrc].split()
        op = [o for o in op if not o.startswith("@")]
        g[3].append(op[0].split(".")[0] if op else "")
    for ex, (n, tex, st, ops) in sorted(groups.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
        c = Counter(ops)
        print(f"  exec={ex:>10} n={n:4d} exec%={tex / tot_ex:5.1%} stall%={st / tot_st:5.1%} ", dict(c.most_common(8)))
