"""Shared-memory wavefronts per CUDA source line (total / excessive) from
`ncu -i REP --page source --csv --print-source cuda,sass`."""
import csv
import sys
from collections import defaultdict


def main(path, top=15):
    rows = list(csv.reader(open(path)))
    cur, hdr = None, None
    wf, ex, text = defaultdict(float), defaultdict(float), {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            iw, ie = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive")
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        key = (cur, int(r[0]))
        text[key] = r[1][:90]
        try:
            wf[key] += float(r[iw] or 0)
            ex[key] += float(r[ie] or 0)
        except (ValueError, IndexError):
            pass
    tw, te = sum(wf.values()) or 1, sum(ex.values())
    print("shared wavefronts %.3e excessive %.3e (%.0f%%)" % (tw, te, 100 * te / tw))
    for k in sorted(wf, key=lambda k: -wf[k])[:top]:
        print("%5.1f%% wf (%4.0f%% excessive)  %s:%d  %s" % (100 * wf[k] / tw, 100 * ex[k] / (wf[k] or 1), k[0], k[1], text[k]))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)
