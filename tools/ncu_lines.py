"""Per-source-line summary of an ncu report (instructions executed, stall samples).

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > mix.csv
    python tools/ncu_lines.py mix.csv [top]

Prints the source lines with the most warp-level instructions executed, their
share of the kernel total, the stall samples, and the opcode mix per line.
"""
import csv
import sys
from collections import Counter, defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    fname = None
    hdr = None
    per_line = defaultdict(lambda: [0, 0, Counter()])
    src_text = {}
    cur = None
    ops = Counter()
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            ie = hdr.index("Instructions Executed")
            st = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) - 5:
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            src_text[cur] = r[1].strip()[:70]
            continue
        if r[2] in ("-", "...") or cur is None:
            continue
        try:
            n = int(r[ie])
            s = int(r[st])
        except ValueError:
            continue
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        op = op.split(".")[0]
        per_line[cur][0] += n
        per_line[cur][1] += s
        per_line[cur][2][op] += n
        ops[op] += n
    tot = sum(v[0] for v in per_line.values())
    tst = sum(v[1] for v in per_line.values())
    print("total warp-instructions %.4g, stall samples %d" % (tot, tst))
    print("opcode mix:", ", ".join("%s %.1f%%" % (k, 100.0 * v / tot) for k, v in ops.most_common(14)))
    for k, v in sorted(per_line.items(), key=lambda kv: -kv[1][0])[:top]:
        mix = " ".join("%s:%d" % (o, c * 100 // max(v[0], 1)) for o, c in v[2].most_common(4))
        print("%5.1f%% %5.1f%%st %s:%d  %-70s %s" % (100.0 * v[0] / tot, 100.0 * v[1] / max(tst, 1),
                                                   k[0], k[1], src_text.get(k, ""), mix))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
