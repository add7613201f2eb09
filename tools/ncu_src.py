"""Summarise an ncu `--page source --csv --print-source cuda,sass` dump:
instructions executed and stall samples per CUDA source line (top N)."""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = None
    cur_file = None
    inst = defaultdict(float)
    samp = defaultdict(float)
    text = {}
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        key = (cur_file, int(r[0]))
        text[key] = r[1][:90]
        try:
            inst[key] += float(r[hdr.index("Instructions Executed")] or 0)
            samp[key] += float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            pass
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    print(f"total inst {ti:.3e}  samples {ts:.0f}")
    for k in sorted(inst, key=lambda k: -inst[k])[:top]:
        print(f"{100*inst[k]/ti:5.1f}% inst {100*samp[k]/ts:5.1f}% stall  {k[0]}:{k[1]}  {text[k]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
