"""Print the key fields of bench JSON lines: python tools/show.py files..."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f, "unreadable", e)
        continue
    r = d.get("roofline") or {}
    print(f, d.get("ms_per_step"), "path", d.get("path_frac"), "dom", r.get("kernel"), r.get("frac"),
          {k: v[0] for k, v in (d.get("kernels") or {}).items()})
