"""Copies one refresh run (tools/refresh_profiles.sh -> gpurun_out/prof) into
profiles/ as the round's artefacts: bench / reference lines, the default
command's ncu launch list and per-kernel shares, the DRAM-traffic table
(csv + the json bench.py reads), the ncu --set full summary and the GPU test
log.    python tools/collect_profiles.py [round-tag, default r02]"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(REPO, "gpurun_out", "prof")
DST = os.path.join(REPO, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"

SHORT = {"k_large_adj2": "large_adj2", "k_large_fwd2": "large_fwd2", "k_large_adj1": "large_adj1",
         "k_large_fwd1_fz": "large_fwd1", "k_dwt_wpyr": "dwt_pyr", "k_wv_adj": "wv_adj",
         "k_wv_fwd": "wv_fwd", "k_normal_rows_reg": "normal_rows", "k_small_fwd": "small_fwd",
         "k_small_adj": "small_adj"}


def last_json_line(path):
    lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
    return lines[-1] if lines else None


def main():
    for c in range(1, 6):
        line = last_json_line(os.path.join(SRC, f"bench_cfg{c}.json"))
        if line:
            open(os.path.join(DST, f"{TAG}_bench_cfg{c}.json"), "w").write(line + "\n")
    for c in (2, 3):
        p = os.path.join(SRC, f"reference_cfg{c}.json")
        if os.path.exists(p) and last_json_line(p):
            open(os.path.join(DST, f"{TAG}_reference_cfg{c}.json"), "w").write(last_json_line(p) + "\n")
    shutil.copy(os.path.join(SRC, "gputest.log"), os.path.join(DST, f"{TAG}_gputest.log"))
    # launch list of the default command + shares of one device step
    shutil.copy(os.path.join(SRC, "launches_cfg3.csv"), os.path.join(DST, f"{TAG}_launches_cfg3.csv"))
    rows = list(csv.reader(open(os.path.join(SRC, "launches_cfg3.csv"))))
    hdr = next(r for r in rows if "Kernel Name" in r)
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    gi = hdr.index("Grid Size")
    body = [r for r in rows[rows.index(hdr) + 2:] if len(r) > vi]
    # full device steps: 13 launches from k_wav_coarse (one CTA per vector of the batch of 32)
    # whose 7th launch is the full-batch k_large_adj2; averaged per kernel over the steps
    per = collections.OrderedDict()
    nsteps = 0
    for i, r in enumerate(body):
        if "k_wav_coarse" in r[ki] and r[gi] == "(32, 1, 1)" and i + 13 <= len(body) and \
                "k_large_adj2" in body[i + 6][ki] and body[i + 6][gi] == "(256, 32, 1)":
            nsteps += 1
            for q in body[i:i + 13]:
                n = q[ki].split("(")[0].replace("void ", "")
                per.setdefault(n, [0.0, 0])
                per[n][0] += float(q[vi])
                per[n][1] += 1
    nsteps = max(nsteps, 1)
    tot = sum(v[0] for v in per.values()) / nsteps
    with open(os.path.join(DST, f"{TAG}_launches_cfg3_shares.csv"), "w") as f:
        f.write("kernel,us_per_step,launches_per_step,share_of_step\n")
        for n, (d, k) in sorted(per.items(), key=lambda kv: -kv[1][0]):
            f.write(f"{n},{d / nsteps / 1000:.1f},{k / nsteps:g},{d / nsteps / tot:.3f}\n")
        f.write(f"total,{tot / 1000:.1f},,1.000\n")
    # DRAM traffic per launch
    shutil.copy(os.path.join(SRC, "ncu_traffic.csv"), os.path.join(DST, f"{TAG}_ncu_traffic.csv"))
    agg = collections.OrderedDict()
    for r in csv.reader(open(os.path.join(SRC, "ncu_traffic.csv"))):
        if len(r) < 16:
            continue
        agg.setdefault((r[0], r[5]), collections.defaultdict(list))[r[-3]].append(float(r[-1]))
    old = json.load(open(os.path.join(DST, f"{TAG}_traffic.json"))) if os.path.exists(os.path.join(DST, f"{TAG}_traffic.json")) else {}
    out = {"source": f"tools/ncu_traffic.sh -> profiles/{TAG}_ncu_traffic.csv: ncu --metrics dram__bytes_read.sum,"
                     "dram__bytes_write.sum on the second call's launches of each config's leading kernels (cold L2 "
                     "per ncu replay); multi-launch kernels: the per-launch average over one step's launches"}
    if "1" in old:
        out["1"] = old["1"]
    for (cfg, kern), m in agg.items():
        c = cfg.replace("cfg", "")
        rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
        per_launch = [a + b for a, b in zip(rd, wr)]
        name = kern.replace("void ", "").split("(")[0]
        short = next((v for k, v in SHORT.items() if name.startswith(k)), name)
        note = f"{name}, {len(per_launch)} launch(es) per call"
        if len(per_launch) > 1:
            note += " (per-launch average of " + " + ".join(f"{x / 1e6:.1f}" for x in per_launch) + " MB)"
        out.setdefault(c, []).append({"kernel": short, "bytes": int(sum(per_launch) / len(per_launch)), "launch": note})
    json.dump(out, open(os.path.join(DST, f"{TAG}_traffic.json"), "w"), indent=1)
    # ncu --set full summary of the strided passes
    for name in ("cfg3_fwd2_adj2", "cfg3_pass1_pyramids", "cfg4_warp_kernels", "cfg5_normal_rows"):
        rep = os.path.join(SRC, name + ".ncu-rep")
        if os.path.exists(rep):
            txt = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_summary.py"), rep],
                                 capture_output=True, text=True).stdout
            open(os.path.join(DST, f"{TAG}_ncu_{name}.txt"), "w").write(txt)
    print(open(os.path.join(DST, f"{TAG}_launches_cfg3_shares.csv")).read())


if __name__ == "__main__":
    main()
