"""Stall samples / instructions per CUDA source line from
`ncu -i REP --page source --csv --print-source cuda,sass --kernel-name regex:K`."""
import csv
import sys
from collections import defaultdict


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur, hdr = None, None
    inst, samp, text = defaultdict(float), defaultdict(float), {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        key = (cur, int(r[0]))
        text[key] = r[1][:100]
        try:
            samp[key] += float(r[4] or 0)
            inst[key] += float(r[7] or 0)
        except (ValueError, IndexError):
            pass
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    print("total inst %.3e samples %.0f" % (ti, ts))
    for k in sorted(samp, key=lambda k: -samp[k])[:top]:
        print("%5.1f%% stall %5.1f%% inst  %s:%d  %s" % (100 * samp[k] / ts, 100 * inst[k] / ti, k[0], k[1], text[k]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
