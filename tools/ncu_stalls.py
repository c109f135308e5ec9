"""Per-source-line stall breakdown of an ncu report's source page.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_stalls.py src.csv stall_long_sb [top]

Prints, for one stall reason (column name of the source page), the source
lines with the most samples of that reason and their share of all samples of
the reason.
"""
import csv
import sys
from collections import defaultdict


def main(path, reason, top=25):
    rows = list(csv.reader(open(path)))
    fname = hdr = cur = None
    per = defaultdict(int)
    text = {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            col = hdr.index(reason)
            continue
        if hdr is None or len(r) < len(hdr) - 5:
            continue
        if r[0]:
            cur = (fname, int(r[0]))
            text[cur] = r[1].strip()[:80]
            continue
        if cur is None:
            continue
        try:
            per[cur] += int(r[col])
        except (ValueError, IndexError):
            pass
    tot = sum(per.values()) or 1
    print(f"{reason}: {tot} samples")
    for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
        print("%5.1f%% %s:%d  %s" % (100.0 * v / tot, k[0], k[1], text.get(k, "")))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
